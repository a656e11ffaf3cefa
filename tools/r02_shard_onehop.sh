# (A/B 8 of profiles/r02_ab_keyset.md; the key-set one-hop kernel it measured was reverted.)
# Round-2: one-hop sharded routers through the key-set scan (kernels.cuh scan_cset_kernel SH 1 / 2):
# sharded parity, the one-hop simulation with the key-set scan (default) and with the older
# scan_shard_kernel (SSPD_CSET=0), the relayed simulation beside it, and the C2 bench as a check.
#   /usr/local/graft/bin/gpurun --timeout 3600 -- 'bash tools/r02_shard_onehop.sh'
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_dist1.py tests/test_gpu_keyset.py tests/test_cpp_api.py -q -k "shard or relay or routers or exchange or keyset or cpp" > gpurun_out/r3g_pytest.log 2>&1
python bench.py --no-cpu-baseline --no-e2e > gpurun_out/r3g_c2.json 2> gpurun_out/r3g_c2.err
for n in 2 4 8; do
  python tools/sim_shard_router.py --routers $n > gpurun_out/r3g_onehop_ks_$n.md 2> gpurun_out/r3g_onehop_ks_$n.err
  SSPD_CSET=0 python tools/sim_shard_router.py --routers $n > gpurun_out/r3g_onehop_ps_$n.md 2> gpurun_out/r3g_onehop_ps_$n.err
  python tools/sim_relay_router.py --routers $n > gpurun_out/r3g_relay_$n.md 2> gpurun_out/r3g_relay_$n.err
done
