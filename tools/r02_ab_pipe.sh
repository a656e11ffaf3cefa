# Round-2 A/B of the C2 scan kernels (run through gpurun):
#   /usr/local/graft/bin/gpurun --timeout 3000 -- 'bash tools/r02_ab_pipe.sh'
# SSPD_DEDUP_PIPE: -1 = round-1 scan_dedup_kernel, 0 = pipelined, 1 = pipelined with L2 eviction
# priorities.  Bench lines, then one ncu --set full capture of each pipelined variant.
mkdir -p gpurun_out
for cfg in c2 c2p64; do
  for v in -1 0 1; do
    SSPD_DEDUP_PIPE=$v python bench.py --config $cfg --no-cpu-baseline --no-e2e > gpurun_out/r2d_${cfg}_pipe$v.json 2> gpurun_out/r2d_${cfg}_pipe$v.err
  done
done
M=smsp__sass_data_bytes_mem_global_op_ld.sum,smsp__sass_data_bytes_mem_global_op_atom.sum,smsp__sass_data_bytes_mem_global_op_red.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_atom_lookup_miss.sum,lts__t_sectors_srcunit_tex_op_atom_lookup_hit.sum
for v in 0 1; do
  SSPD_DEDUP_PIPE=$v ncu --set full --metrics $M --clock-control none --import-source on -k regex:scan_dedup -s 3 -c 1 -f \
    -o gpurun_out/r2d_c2_scan_pipe$v python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2d_ncu_pipe$v.log 2>&1
done
