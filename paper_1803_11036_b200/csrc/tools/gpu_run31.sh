./tools/bin/bench_api > gpurun_out/bench_api.md 2>&1
python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "scan or batch or update" > gpurun_out/pytest_gpu_quick.log 2>&1
