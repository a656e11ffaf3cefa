python -m pytest tests/test_gpu_narrow.py -q -x > gpurun_out/pytest_narrow.log 2>&1
for w in 8 16 32; do
  python bench.py --stamp-width $w --steps 10 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/c2_w$w.json 2> gpurun_out/c2_w$w.err
done
