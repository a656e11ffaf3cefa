python -m pytest tests/test_gpu_parity.py -q -x -k "extreme" > gpurun_out/pytest_extreme.log 2>&1
