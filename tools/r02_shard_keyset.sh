# (A/B 7 of profiles/r02_ab_keyset.md; the shard key-set code it measured was reverted.)
# Round-2: the sharded routers' scans with compact key sets (kernels.cuh scan_shard_kernel KS = 1) --
# parity of the sharded/relayed paths on one device, then the one-GPU router-slot simulation at
# N = 2, 4, 8 with key sets (default) and with the 8-byte pair sets (SSPD_CSET=0).
#   /usr/local/graft/bin/gpurun --timeout 3000 -- 'bash tools/r02_shard_keyset.sh'
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py -q -k "shard or relay or routers" > gpurun_out/r3c_pytest_shard.log 2>&1
python -m pytest tests/test_gpu_dist1.py tests/test_cpp_api.py -q > gpurun_out/r3c_pytest_dist1_cpp.log 2>&1
for n in 2 4 8; do
  python tools/sim_relay_router.py --routers $n > gpurun_out/r3c_sim_ks_$n.md 2> gpurun_out/r3c_sim_ks_$n.err
  SSPD_CSET=0 python tools/sim_relay_router.py --routers $n > gpurun_out/r3c_sim_ps_$n.md 2> gpurun_out/r3c_sim_ps_$n.err
done
