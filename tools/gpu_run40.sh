for f in 1 0; do
  echo "== c1 direct filter $f" >> gpurun_out/ab_c1_filter.txt
  python bench.py --config c1 --scan-mode direct --filter $f --steps 20 --warmup 3 --no-cpu-baseline >> gpurun_out/ab_c1_filter.txt 2>&1
done
for f in 1 0; do
  echo "== c2 direct filter $f" >> gpurun_out/ab_c1_filter.txt
  python bench.py --config c2 --scan-mode direct --filter $f --steps 10 --warmup 3 --no-cpu-baseline --no-e2e >> gpurun_out/ab_c1_filter.txt 2>&1
done
