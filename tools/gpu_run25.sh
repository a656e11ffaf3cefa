CMD="python bench.py --no-cpu-baseline"
$CMD > gpurun_out/ncu7_plain.json 2> gpurun_out/ncu7_plain.err && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ncu7_launches.csv $CMD > gpurun_out/ncu7_launches.log 2>&1
CMD2="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
$CMD2 > gpurun_out/ncu8_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"scan_dedup|finalize_count|hot_mark|hot_write|level" -c 6 -o gpurun_out/ncu8_full $CMD2 > gpurun_out/ncu8_full.log 2>&1
echo done
