python bench.py --stamp-width 16 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/w16_plain.json 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:scan_narrow -s 3 -c 1 -f -o gpurun_out/w16_scan python bench.py --stamp-width 16 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/w16_ncu.log 2>&1
