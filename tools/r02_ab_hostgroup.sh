# Round-2 A/B: host-grouped pair set with 256-bit sector probes (-DSSPD_PIPE_SECT=2; a cip's pairs in one
# 32-slot group), variants v/w/x in variants/, at the default 2^25-entry set and a 2^26 one.
#   /usr/local/graft/bin/gpurun --timeout 2400 -- 'bash tools/r02_ab_hostgroup.sh'
mkdir -p gpurun_out
for cfg in c2 c2p64; do
  python bench.py --config $cfg --no-cpu-baseline --no-e2e > gpurun_out/r2m_${cfg}_a.json 2> gpurun_out/r2m_${cfg}_a.err
  for n in v w x; do
    SSPD_LIB=$PWD/variants/libsspd_cuda_$n.so python bench.py --config $cfg --no-cpu-baseline --no-e2e > gpurun_out/r2m_${cfg}_$n.json 2> gpurun_out/r2m_${cfg}_$n.err
    SSPD_PAIRSET_LOG2=26 SSPD_LIB=$PWD/variants/libsspd_cuda_$n.so python bench.py --config $cfg --no-cpu-baseline --no-e2e > gpurun_out/r2m_${cfg}_${n}26.json 2> gpurun_out/r2m_${cfg}_${n}26.err
  done
done
M=lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_atom_lookup_miss.sum,lts__t_sectors_srcunit_tex_op_atom_lookup_hit.sum
SSPD_PAIRSET_LOG2=26 SSPD_LIB=$PWD/variants/libsspd_cuda_w.so ncu --set full --metrics $M --clock-control none -k regex:scan_dedup -s 3 -c 1 -f \
    -o gpurun_out/r2m_c2_scan_w26 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2m_ncu_w26.log 2>&1
