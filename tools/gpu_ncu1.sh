CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/ncu1_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ncu1_launches.csv $CMD > gpurun_out/ncu1_launches.log 2>&1
$CMD > gpurun_out/ncu1_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"scan_bitmap|commit_kernel|finalize_kernel" -c 3 -o gpurun_out/ncu1_full $CMD > gpurun_out/ncu1_full.log 2>&1
echo exit $?
