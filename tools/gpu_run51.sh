python bench.py --config c1 --steps 20 --no-cpu-baseline > gpurun_out/c1_chunk.json 2>&1
python bench.py --steps 10 --no-cpu-baseline > gpurun_out/c2_chunk.json 2>&1
