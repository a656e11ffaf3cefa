python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1
python bench.py --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/ncu2_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"scan_bitmap|commit_kernel" -c 2 -o gpurun_out/ncu2_full $CMD > gpurun_out/ncu2_full.log 2>&1
echo done
