echo "== base" >> gpurun_out/ab12.log
python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e >> gpurun_out/ab12.log 2>&1
for v in c0 c1k c4k; do
echo "== $v" >> gpurun_out/ab12.log
SSPD_LIB=$PWD/variants/libsspd_cuda_$v.so python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e >> gpurun_out/ab12.log 2>&1
done
