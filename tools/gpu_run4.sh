python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1
for mode in dedup bitmap; do
  echo "== c2 $mode" >> gpurun_out/ab2.log
  python bench.py --steps 5 --warmup 3 --no-cpu-baseline --scan-mode $mode >> gpurun_out/ab2.log 2>&1
done
echo "== c1 auto" >> gpurun_out/ab2.log
python bench.py --config c1 --steps 5 --warmup 3 --no-cpu-baseline >> gpurun_out/ab2.log 2>&1
echo "== c1 dedup" >> gpurun_out/ab2.log
python bench.py --config c1 --steps 5 --warmup 3 --no-cpu-baseline --scan-mode dedup >> gpurun_out/ab2.log 2>&1
