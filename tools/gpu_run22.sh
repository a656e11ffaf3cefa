for v in batchppt2 batchppt2minb5 ppt2 batchppt2bps4; do
echo "== $v" >> gpurun_out/ab11.log
SSPD_LIB=$PWD/variants/libsspd_cuda_$v.so python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e >> gpurun_out/ab11.log 2>&1
done
echo "== base" >> gpurun_out/ab11.log
python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e >> gpurun_out/ab11.log 2>&1
