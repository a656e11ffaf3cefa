python -m pytest tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1
for mode in dedup binned; do
echo "== c2 $mode" >> gpurun_out/ab7.log
python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --scan-mode $mode >> gpurun_out/ab7.log 2>&1
done
