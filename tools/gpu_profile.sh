# The profiles/ evidence for the C2 scan (run through gpurun; one profiler per call is fine here
# because each ncu run follows the same command exiting 0 without it):
#   /usr/local/graft/bin/gpurun --timeout 2400 -- 'bash tools/gpu_profile.sh'
# then: python tools/ncu_summary.py launches gpurun_out/launches_c2.csv
#       python tools/ncu_summary.py full gpurun_out/c2_scan.ncu-rep
set -e
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/c2_plain.json 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c2.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1
ncu --set full --metrics smsp__sass_data_bytes_mem_global_op_ld.sum,smsp__sass_data_bytes_mem_global_op_atom.sum,smsp__sass_data_bytes_mem_global_op_red.sum \
    --clock-control none --import-source on -k regex:scan_dedup -s 3 -c 1 -f -o gpurun_out/c2_scan \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full.log 2>&1
