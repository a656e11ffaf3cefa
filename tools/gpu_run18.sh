echo "== base" >> gpurun_out/ab9.log
python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e >> gpurun_out/ab9.log 2>&1
for v in ppt8 minb6 ppt8minb4 bps4 bps16; do
echo "== $v" >> gpurun_out/ab9.log
SSPD_LIB=$PWD/variants/libsspd_cuda_$v.so python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e >> gpurun_out/ab9.log 2>&1
done
