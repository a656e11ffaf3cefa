# Round-2 final evidence (same steps as tools/r02_keyset_verify.sh, outputs ${TAG}_* (TAG defaults to r3i)):
#   /usr/local/graft/bin/gpurun --timeout 3600 -- 'bash tools/r02_final_verify.sh'
# GPU tests, smoke, bench lines (C2 with the CPU reference and e2e, C2 64-entry pools, C1), then the
# launch list and one ncu --set full capture of the scan per Zipf config -- each ncu run after the
# same command exited 0 without ncu.
TAG=${TAG:-r3i}
mkdir -p gpurun_out
python -m pytest tests -q -m gpu > gpurun_out/${TAG}_pytest_gpu.log 2>&1
python -c "import __graft_entry__ as G; G.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
python bench.py > gpurun_out/${TAG}_bench_c2.json 2> gpurun_out/${TAG}_bench_c2.err
python bench.py --config c2p64 --no-cpu-baseline > gpurun_out/${TAG}_bench_c2p64.json 2> gpurun_out/${TAG}_bench_c2p64.err
python bench.py --config c1 > gpurun_out/${TAG}_bench_c1.json 2> gpurun_out/${TAG}_bench_c1.err
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_c2_plain.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches_c2.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_ncu_launches.log 2>&1
M=smsp__sass_data_bytes_mem_global_op_ld.sum,smsp__sass_data_bytes_mem_global_op_atom.sum,smsp__sass_data_bytes_mem_global_op_red.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_atom_lookup_miss.sum,lts__t_sectors_srcunit_tex_op_atom_lookup_hit.sum
for cfg in c2 c2p64; do
  ncu --set full --metrics $M --clock-control none --import-source on -k regex:scan_cset -s 3 -c 1 -f \
    -o gpurun_out/${TAG}_${cfg}_scan python bench.py --config $cfg --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_ncu_$cfg.log 2>&1
done
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${TAG}_bench_ref.json 2> gpurun_out/${TAG}_bench_ref.err
