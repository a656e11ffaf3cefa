python -m pytest tests/test_gpu_parity.py tests/test_synth.py -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1
python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ab6.log 2>&1
python bench.py --config c1 --steps 10 --warmup 3 --no-cpu-baseline --scan-mode dedup >> gpurun_out/ab6.log 2>&1
