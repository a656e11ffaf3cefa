# Round-2 A/B #5 of the key-set scan: the pair stream loaded one iteration ahead (pf, -DSSPD_CSET_PF=1)
# and 3 CTAs/SM without register cap pressure (m3, -DSSPD_PIPE_MINB=3; pf_m3 both).
#   /usr/local/graft/bin/gpurun --timeout 2400 -- 'bash tools/r02_ab_cset5.sh'
mkdir -p gpurun_out
run() {  # name, env...
  local name=$1; shift
  for cfg in c2 c2p64; do
    env "$@" python bench.py --config $cfg --no-cpu-baseline --no-e2e > gpurun_out/r2z_${cfg}_$name.json 2> gpurun_out/r2z_${cfg}_$name.err
  done
}
V=$PWD/variants
run default SSPD_CSET=1
run pf SSPD_LIB=$V/libsspd_cuda_pf.so
run m3 SSPD_LIB=$V/libsspd_cuda_m3.so
run pf_m3 SSPD_LIB=$V/libsspd_cuda_pf_m3.so
run default_b SSPD_CSET=1
