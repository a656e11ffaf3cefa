python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1
