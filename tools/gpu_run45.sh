for m in dedup split; do
  echo "== c2 $m" >> gpurun_out/ab_split.txt
  python bench.py --scan-mode $m --steps 10 --no-cpu-baseline --no-e2e >> gpurun_out/ab_split.txt 2>&1
done
python -m pytest tests/test_gpu_parity.py -q -x -k "split" > gpurun_out/pytest_split.log 2>&1
