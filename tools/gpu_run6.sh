python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/ncu3_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"scan_dedup" -c 1 -o gpurun_out/ncu3_full $CMD > gpurun_out/ncu3_full.log 2>&1
echo done
