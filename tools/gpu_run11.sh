timeout 1200 compute-sanitizer --tool memcheck --leak-check no --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -x -q -k "desk or invariance or update or finalize or overflow or merge or cells or repeated or window" > gpurun_out/memcheck.log 2>&1
echo "exit $?" >> gpurun_out/memcheck.log
