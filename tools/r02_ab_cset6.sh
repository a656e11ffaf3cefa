# Round-2 A/B #6 of the key-set scan: 2 or 4 passes over each batch, each pass taking only the keys
# homed in its 1/passes of the set (so a pass probes 32 MiB / 16 MiB of the 64 MiB set), against
# one pass.  The pair stream is read once per pass.
#   /usr/local/graft/bin/gpurun --timeout 2400 -- 'bash tools/r02_ab_cset6.sh'
mkdir -p gpurun_out
python -m pytest tests/test_gpu_keyset.py -q -k "bit_exact or distinct" > gpurun_out/r3a_pytest_keyset.log 2>&1
run() {  # name, env...
  local name=$1; shift
  for cfg in c2 c2p64; do
    env "$@" python bench.py --config $cfg --no-cpu-baseline --no-e2e > gpurun_out/r3a_${cfg}_$name.json 2> gpurun_out/r3a_${cfg}_$name.err
  done
}
run p1 SSPD_CSET_PASSES=1
run p2 SSPD_CSET_PASSES=2
run p4 SSPD_CSET_PASSES=4
run p1_b SSPD_CSET_PASSES=1
