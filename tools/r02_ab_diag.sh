# Round-2 A/B #12, a cost split of the key-set scan with diagnostic builds (their results are wrong;
# timing only): variants/libsspd_cuda_diag1.so skips the window-ring moves, diag2 also stamps with
# non-returning red.max, diag3 keeps the returning stamps but drops the ring moves.  Build them with
#   nvcc <the Makefile's NVFLAGS> -DSSPD_AB_DIAG={1,2,3} -shared -o variants/libsspd_cuda_diag{1,2,3}.so paper_1803_11036_b200/csrc/sspd_cuda.cu -lgomp
#   /usr/local/graft/bin/gpurun --timeout 1800 -- 'bash tools/r02_ab_diag.sh'
mkdir -p gpurun_out
T=${TAG:-r4i}
run() {  # name, env...
  local name=$1; shift
  for cfg in c2 c2p64; do
    timeout 600 env "$@" python bench.py --config $cfg --no-cpu-baseline --no-e2e > gpurun_out/${T}_${cfg}_$name.json 2> gpurun_out/${T}_${cfg}_$name.err
  done
}
run base
run noring SSPD_LIB=$PWD/variants/libsspd_cuda_diag1.so
run redstamps SSPD_LIB=$PWD/variants/libsspd_cuda_diag2.so
run retnoring SSPD_LIB=$PWD/variants/libsspd_cuda_diag3.so
run base_b
for v in 3; do
  SSPD_LIB=$PWD/variants/libsspd_cuda_diag$v.so ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_op_read_hit_rate.pct,lts__t_sectors_srcunit_tex_op_red.sum,lts__t_sectors_srcunit_tex_op_atom.sum \
    --clock-control none -k regex:scan_cset -s 3 -c 1 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${T}_ncu_diag$v.log 2>&1
  grep -E "gpu__time|dram__bytes|hit_rate|op_red|op_atom" gpurun_out/${T}_ncu_diag$v.log
done
