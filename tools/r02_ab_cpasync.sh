# Round-2 A/B: the pipelined scan's pair stream through cp.async into a per-thread shared-memory double
# buffer (-DSSPD_PIPE_CPASYNC=1; y: MINB 4, z: MINB 3), variants in variants/; then parity with y.
#   /usr/local/graft/bin/gpurun --timeout 2400 -- 'bash tools/r02_ab_cpasync.sh'
mkdir -p gpurun_out
for cfg in c2 c2p64; do
  python bench.py --config $cfg --no-cpu-baseline --no-e2e > gpurun_out/r2n_${cfg}_a.json 2> gpurun_out/r2n_${cfg}_a.err
  for n in y z; do
    SSPD_LIB=$PWD/variants/libsspd_cuda_$n.so python bench.py --config $cfg --no-cpu-baseline --no-e2e > gpurun_out/r2n_${cfg}_$n.json 2> gpurun_out/r2n_${cfg}_$n.err
  done
  python bench.py --config $cfg --no-cpu-baseline --no-e2e > gpurun_out/r2n_${cfg}_a2.json 2> gpurun_out/r2n_${cfg}_a2.err
done
SSPD_LIB=$PWD/variants/libsspd_cuda_y.so python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -q -m gpu -x -k "dedup or auto or window or fuzz or async or readbacks" > gpurun_out/r2n_tests_y.log 2>&1
