# Round-2 A/B #4 of the key set: the bucket walk's limit and code shape (4-entry buckets, 2^24,
# L2 priorities).  default = 8 buckets unrolled, then up to 48 in a loop of its own; lim8 = one loop
# of 8 (A/B 3's kernel); lim8b = the default shape with limit 8; lim48inl = one loop of 48;
# far1 = buckets past the home one in a non-inlined function.
#   /usr/local/graft/bin/gpurun --timeout 2400 -- 'bash tools/r02_ab_cset4.sh'
mkdir -p gpurun_out
run() {  # name, env...
  local name=$1; shift
  for cfg in c2 c2p64; do
    env "$@" python bench.py --config $cfg --no-cpu-baseline --no-e2e > gpurun_out/r2x_${cfg}_$name.json 2> gpurun_out/r2x_${cfg}_$name.err
  done
}
V=$PWD/variants
run default SSPD_CSET=1
run lim8 SSPD_LIB=$V/libsspd_cuda_lim8.so
run lim8b SSPD_LIB=$V/libsspd_cuda_lim8b.so
run lim48inl SSPD_LIB=$V/libsspd_cuda_lim48inl.so
run far1 SSPD_LIB=$V/libsspd_cuda_far1.so
run default_b SSPD_CSET=1
