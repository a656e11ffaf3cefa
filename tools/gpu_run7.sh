python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1
for lg in 22 23 24 25; do
  echo "== c2 dedup log2=$lg" >> gpurun_out/ab4.log
  SSPD_PAIRSET_LOG2=$lg python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e >> gpurun_out/ab4.log 2>&1
done
for lg in 23 24; do for mb in 64 96; do
  echo "== c2 dedup log2=$lg persist=$mb" >> gpurun_out/ab4.log
  SSPD_L2_PERSIST=$mb SSPD_PAIRSET_LOG2=$lg python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e >> gpurun_out/ab4.log 2>&1
done; done
python -c "import torch; p=torch.cuda.get_device_properties(0); print(p)" >> gpurun_out/ab4.log 2>&1
