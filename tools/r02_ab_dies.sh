# Round-2 A/B #11 of the key-set scan (rejected; the kernels are in profiles/r02_ab_dies.patch -- apply it first): the set split between the B200's two dies ($SSPD_CSET_DIES=1:
# cset_bin_kernel puts each pair on the list of the die owning its key's part of the set, and each die's
# CTAs scan their own list) against the default scan.  Die probe and parity first.
#   /usr/local/graft/bin/gpurun --timeout 2400 -- 'bash tools/r02_ab_dies.sh'
mkdir -p gpurun_out
T=${TAG:-r4g}
timeout 300 ./tools/bin/die_probe > gpurun_out/${T}_die_probe.txt 2>&1
SSPD_DIES_VERBOSE=1 timeout 900 python -m pytest tests/test_gpu_keyset.py -q -x -k "dies" > gpurun_out/${T}_pytest_dies.log 2>&1
tail -2 gpurun_out/${T}_pytest_dies.log
run() {  # name, env...
  local name=$1; shift
  for cfg in c2 c2p64; do
    timeout 600 env "$@" python bench.py --config $cfg --no-cpu-baseline --no-e2e > gpurun_out/${T}_${cfg}_$name.json 2> gpurun_out/${T}_${cfg}_$name.err
  done
}
run base
run dies SSPD_CSET_DIES=1 SSPD_DIES_VERBOSE=1
run base_b
run dies_b SSPD_CSET_DIES=1
SSPD_CSET_DIES=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_op_read_hit_rate.pct,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread \
  --clock-control none -k regex:"cset_" -s 6 -c 4 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${T}_ncu_dies.log 2>&1
grep -E "cset_|gpu__time|dram__bytes|hit_rate|warps_active|registers" gpurun_out/${T}_ncu_dies.log | head -40
grep -h "dies:" gpurun_out/${T}_*.err | sort | uniq -c
