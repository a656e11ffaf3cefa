# Round-2 A/B: resident CTAs per SM for the scan kernels sized by SSPD_SCAN_BLOCKS_PER_SM (direct, dedup,
# sharded; the key-set scan has its own): 4 (default) vs 6 and 8 -- C1 bench and the N = 2 / 8
# router-slot simulation.
#   /usr/local/graft/bin/gpurun --timeout 2400 -- 'bash tools/r02_ab_bps.sh'
mkdir -p gpurun_out
V=$PWD/variants
for b in 4 6 8; do
  if [ $b = 4 ]; then L=""; else L="SSPD_LIB=$V/libsspd_cuda_bps$b.so"; fi
  env $L python bench.py --config c1 --no-cpu-baseline --no-e2e > gpurun_out/r3e_c1_bps$b.json 2> gpurun_out/r3e_c1_bps$b.err
  for n in 2 8; do
    env $L python tools/sim_relay_router.py --routers $n > gpurun_out/r3e_sim_bps${b}_$n.md 2> gpurun_out/r3e_sim_bps${b}_$n.err
  done
done
