python bench.py --config c1 --steps 20 --no-cpu-baseline > gpurun_out/c1_pool.json 2>&1
python bench.py --steps 10 --no-cpu-baseline --no-e2e > gpurun_out/c2_pool.json 2>&1
