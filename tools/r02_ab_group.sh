# Round-2 A/B: pair set hashed by cip (a host's pairs in one 128 B line; -DSSPD_PAIR_GROUP=1) with
# probe limits 8/16/24 (variants i/j/k, built into variants/), then parity with it.
#   /usr/local/graft/bin/gpurun --timeout 2400 -- 'bash tools/r02_ab_group.sh'
mkdir -p gpurun_out
for cfg in c2 c2p64; do
  python bench.py --config $cfg --no-cpu-baseline --no-e2e > gpurun_out/r2g_${cfg}_a.json 2> gpurun_out/r2g_${cfg}_a.err
  for n in i j k; do
    SSPD_LIB=$PWD/variants/libsspd_cuda_$n.so python bench.py --config $cfg --no-cpu-baseline --no-e2e > gpurun_out/r2g_${cfg}_$n.json 2> gpurun_out/r2g_${cfg}_$n.err
  done
  SSPD_PAIRSET_LOG2=26 SSPD_LIB=$PWD/variants/libsspd_cuda_j.so python bench.py --config $cfg --no-cpu-baseline --no-e2e > gpurun_out/r2g_${cfg}_j26.json 2> gpurun_out/r2g_${cfg}_j26.err
done
SSPD_LIB=$PWD/variants/libsspd_cuda_j.so python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_narrow.py -q -m gpu -x -k "dedup or auto or window or fuzz or async or readbacks or shard or narrow" > gpurun_out/r2g_tests_j.log 2>&1
M=lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_atom_lookup_miss.sum,lts__t_sectors_srcunit_tex_op_atom_lookup_hit.sum
SSPD_LIB=$PWD/variants/libsspd_cuda_j.so ncu --set full --metrics $M --clock-control none --import-source on -k regex:scan_dedup -s 3 -c 1 -f \
    -o gpurun_out/r2g_c2_scan_j python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2g_ncu_j.log 2>&1
