# Round-2 A/B of the pipelined scan's occupancy (pairs per thread x CTAs per SM), variants built
# into variants/ (git-ignored) with -DSSPD_PIPE_MINB / -DSSPD_PIPE_PPT:
#   /usr/local/graft/bin/gpurun --timeout 2400 -- 'bash tools/r02_ab_occupancy.sh'
mkdir -p gpurun_out
python bench.py --no-cpu-baseline --no-e2e > gpurun_out/r2f_c2_a.json 2> gpurun_out/r2f_c2_a.err
for n in b c d e f g h; do
  SSPD_LIB=$PWD/variants/libsspd_cuda_$n.so python bench.py --no-cpu-baseline --no-e2e > gpurun_out/r2f_c2_$n.json 2> gpurun_out/r2f_c2_$n.err
done
python bench.py --no-cpu-baseline --no-e2e > gpurun_out/r2f_c2_a2.json 2> gpurun_out/r2f_c2_a2.err
