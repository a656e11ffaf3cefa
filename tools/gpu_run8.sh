for mode in bitmap direct dedup; do
  echo "== c1 $mode" >> gpurun_out/ab5.log
  python bench.py --config c1 --steps 10 --warmup 3 --no-cpu-baseline --scan-mode $mode >> gpurun_out/ab5.log 2>&1
done
CMD="python bench.py --config c1 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --scan-mode bitmap"
$CMD > gpurun_out/ncu4_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"commit_kernel|scan_bitmap" -c 2 -o gpurun_out/ncu4_full $CMD > gpurun_out/ncu4_full.log 2>&1
echo done
