for mode in dedup auto; do
  echo "== c2 $mode" >> gpurun_out/ab3.log
  python bench.py --steps 5 --warmup 3 --no-cpu-baseline --scan-mode $mode >> gpurun_out/ab3.log 2>&1
done
echo "== c1 dedup" >> gpurun_out/ab3.log
python bench.py --config c1 --steps 5 --warmup 3 --no-cpu-baseline --scan-mode dedup >> gpurun_out/ab3.log 2>&1
