SSPD_LIB=$PWD/variants/libsspd_cuda_nostamp.so python bench.py --steps 10 --no-cpu-baseline --no-e2e > gpurun_out/nostamp.json 2>&1
python bench.py --steps 10 --no-cpu-baseline --no-e2e > gpurun_out/stamp.json 2>&1
