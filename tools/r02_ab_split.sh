# Round-2 A/B #10 of the key-set scan (rejected; the kernels are in profiles/r02_ab_split.patch -- apply it first): probe and stamping as two kernels ($SSPD_CSET_SPLIT=1:
# cset_probe_kernel appends fresh keys to per-warp lists, cset_stamp_kernel stamps them) against the
# fused pipelined scan_cset_kernel.  Parity first (key-set suite with the split variants).
#   /usr/local/graft/bin/gpurun --timeout 2400 -- 'bash tools/r02_ab_split.sh'
mkdir -p gpurun_out
T=${TAG:-r4c}
python -m pytest tests/test_gpu_keyset.py -q -k "split" > gpurun_out/${T}_pytest_split.log 2>&1
tail -2 gpurun_out/${T}_pytest_split.log
run() {  # name, env...
  local name=$1; shift
  for cfg in c2 c2p64; do
    env "$@" python bench.py --config $cfg --no-cpu-baseline --no-e2e > gpurun_out/${T}_${cfg}_$name.json 2> gpurun_out/${T}_${cfg}_$name.err
  done
}
run fused
run split SSPD_CSET_SPLIT=1
run fused_b
run split_b SSPD_CSET_SPLIT=1
SSPD_CSET_SPLIT=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_op_read_hit_rate.pct,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread \
  --clock-control none -k regex:cset_ -s 6 -c 4 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${T}_ncu_split.log 2>&1
grep -E "cset_|gpu__time|dram__bytes|hit_rate|warps_active|registers" gpurun_out/${T}_ncu_split.log | head -40
