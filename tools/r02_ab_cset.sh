# Round-2 A/B of the compact key set (kernels.cuh scan_cset_kernel) against the pipelined
# 8-byte pair set (run through gpurun):
#   /usr/local/graft/bin/gpurun --timeout 3000 -- 'bash tools/r02_ab_cset.sh'
# SSPD_CSET=0: scan_dedup_pipe_kernel (the previous default); 1: the key set at 2^SSPD_CSET_LOG2
# entries; SSPD_DEDUP_PIPE=1 adds L2 eviction priorities (set evict_last, stamps evict_first).
mkdir -p gpurun_out
python -m pytest tests/test_gpu_keyset.py -q -x > gpurun_out/r2r_pytest_keyset.log 2>&1
run() {  # name, env...
  local name=$1; shift
  for cfg in c2 c2p64; do
    env "$@" python bench.py --config $cfg --no-cpu-baseline --no-e2e > gpurun_out/r2r_${cfg}_$name.json 2> gpurun_out/r2r_${cfg}_$name.err
  done
}
run pairset SSPD_CSET=0
run cset24 SSPD_CSET=1 SSPD_CSET_LOG2=24
run cset24h SSPD_CSET=1 SSPD_CSET_LOG2=24 SSPD_DEDUP_PIPE=1
run cset25 SSPD_CSET=1 SSPD_CSET_LOG2=25
run cset25h SSPD_CSET=1 SSPD_CSET_LOG2=25 SSPD_DEDUP_PIPE=1
run pairset_b SSPD_CSET=0
M=lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_atom_lookup_miss.sum,lts__t_sectors_srcunit_tex_op_atom_lookup_hit.sum
for v in 0 1; do
  SSPD_CSET=1 SSPD_DEDUP_PIPE=$v ncu --set full --metrics $M --clock-control none --import-source on -k regex:scan_cset -s 3 -c 1 -f \
    -o gpurun_out/r2r_c2_cset_h$v python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2r_ncu_h$v.log 2>&1
done
