echo "== base" >> gpurun_out/ab13.log
python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e >> gpurun_out/ab13.log 2>&1
for v in pf pf4 ppt4; do
echo "== $v" >> gpurun_out/ab13.log
SSPD_LIB=$PWD/variants/libsspd_cuda_$v.so python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e >> gpurun_out/ab13.log 2>&1
done
