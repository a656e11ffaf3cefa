# Round-2 A/B of the pipelined C2 scan's front set (SSPD_FRONT_LOG2; 0 = none), then parity with it on.
#   /usr/local/graft/bin/gpurun --timeout 3000 -- 'bash tools/r02_ab_front.sh'
mkdir -p gpurun_out
for cfg in c2 c2p64; do
  for f in 0 22 23 24; do
    SSPD_FRONT_LOG2=$f python bench.py --config $cfg --no-cpu-baseline --no-e2e > gpurun_out/r2e_${cfg}_front$f.json 2> gpurun_out/r2e_${cfg}_front$f.err
  done
done
for f in 16 23; do
  SSPD_FRONT_LOG2=$f python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -q -m gpu -x -k "dedup or auto or window or fuzz or async or readbacks" > gpurun_out/r2e_tests_front$f.log 2>&1
done
SSPD_FRONT_LOG2=23 python -m pytest tests/test_gpu_fullsize.py -q > gpurun_out/r2e_full.log 2>&1
