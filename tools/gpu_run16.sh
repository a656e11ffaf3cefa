python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1
python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ab8.log 2>&1
python bench.py --config c1 --steps 10 --warmup 3 --no-cpu-baseline >> gpurun_out/ab8.log 2>&1
