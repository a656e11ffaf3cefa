# Round-2 profiles/ evidence (run through gpurun; each ncu run follows the same command exiting 0 without it):
#   /usr/local/graft/bin/gpurun --timeout 2400 -- 'bash tools/r02_profile.sh'
set -e
mkdir -p gpurun_out
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r2k_c2_plain.json 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2k_launches_c2.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r2k_ncu_launches.log 2>&1
M=smsp__sass_data_bytes_mem_global_op_ld.sum,smsp__sass_data_bytes_mem_global_op_atom.sum,smsp__sass_data_bytes_mem_global_op_red.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_atom_lookup_miss.sum,lts__t_sectors_srcunit_tex_op_atom_lookup_hit.sum
python bench.py --config c2p64 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2k_c2p64_plain.json 2>&1
ncu --set full --metrics $M --clock-control none --import-source on -k regex:scan_dedup -s 3 -c 1 -f \
    -o gpurun_out/r2k_c2p64_scan python bench.py --config c2p64 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2k_ncu_c2p64.log 2>&1
python bench.py --config c1 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2k_c1_plain.json 2>&1
ncu --set full --metrics $M --clock-control none --import-source on -k regex:scan_direct -s 3 -c 1 -f \
    -o gpurun_out/r2k_c1_scan python bench.py --config c1 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2k_ncu_c1.log 2>&1
