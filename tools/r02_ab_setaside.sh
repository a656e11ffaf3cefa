# Round-2 A/B #9 of the key-set scan: the persisting-L2 set-aside (cudaLimitPersistingL2CacheSize,
# $SSPD_L2_SETASIDE_MIB) that the set's evict_last probes may occupy, against the driver default 0.
#   /usr/local/graft/bin/gpurun --timeout 2400 -- 'bash tools/r02_ab_setaside.sh'
mkdir -p gpurun_out
run() {  # name, env...
  local name=$1; shift
  for cfg in c2 c2p64; do
    env "$@" python bench.py --config $cfg --no-cpu-baseline --no-e2e > gpurun_out/r4b_${cfg}_$name.json 2> gpurun_out/r4b_${cfg}_$name.err
  done
}
run base
run sa32 SSPD_L2_SETASIDE_MIB=32
run sa64 SSPD_L2_SETASIDE_MIB=64
run sa80 SSPD_L2_SETASIDE_MIB=80
run sa128 SSPD_L2_SETASIDE_MIB=128
run base_b
grep -h "set-aside" gpurun_out/r4b_c2_sa*.err | sort | uniq -c
