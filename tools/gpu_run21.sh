echo "== base" >> gpurun_out/ab10.log
python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e >> gpurun_out/ab10.log 2>&1
for v in batch batchppt2; do
echo "== $v" >> gpurun_out/ab10.log
SSPD_LIB=$PWD/variants/libsspd_cuda_$v.so python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e >> gpurun_out/ab10.log 2>&1
done
