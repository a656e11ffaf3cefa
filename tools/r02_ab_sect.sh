# Round-2 A/B: pair-set probes as 256-bit sector loads (-DSSPD_PIPE_SECT=1), variants l..p in variants/.
#   /usr/local/graft/bin/gpurun --timeout 2400 -- 'bash tools/r02_ab_sect.sh'
mkdir -p gpurun_out
for cfg in c2 c2p64; do
  python bench.py --config $cfg --no-cpu-baseline --no-e2e > gpurun_out/r2h_${cfg}_a.json 2> gpurun_out/r2h_${cfg}_a.err
  for n in l m n o p; do
    SSPD_LIB=$PWD/variants/libsspd_cuda_$n.so python bench.py --config $cfg --no-cpu-baseline --no-e2e > gpurun_out/r2h_${cfg}_$n.json 2> gpurun_out/r2h_${cfg}_$n.err
  done
done
for n in l m; do
SSPD_LIB=$PWD/variants/libsspd_cuda_$n.so python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -q -m gpu -x -k "dedup or auto or window or fuzz or async or readbacks" > gpurun_out/r2h_tests_$n.log 2>&1
done
