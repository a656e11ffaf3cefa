python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1
for cfg in c2 c1; do for mode in bitmap direct; do for f in 0 1; do
  echo "== $cfg $mode filter=$f" >> gpurun_out/ab1.log
  python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --scan-mode $mode --filter $f >> gpurun_out/ab1.log 2>&1
done; done; done
