# Round-2 A/B #3 of the compact key set: bucketized probes (one 16 B / 32 B load per probe) vs
# linear probing by slot, at 2^25 / 2^26 entries.  Default build = 4-entry buckets;
# variants/libsspd_cuda_bw1.so = slot probing (A/B #1-2), bw8 = 8-entry buckets.
#   /usr/local/graft/bin/gpurun --timeout 3000 -- 'bash tools/r02_ab_cset3.sh'
mkdir -p gpurun_out
python -m pytest tests/test_gpu_keyset.py -q > gpurun_out/r2t_pytest_keyset.log 2>&1
SSPD_LIB=$PWD/variants/libsspd_cuda_bw8.so python -m pytest tests/test_gpu_keyset.py -q > gpurun_out/r2t_pytest_keyset_bw8.log 2>&1
run() {  # name, env...
  local name=$1; shift
  for cfg in c2 c2p64; do
    env "$@" python bench.py --config $cfg --no-cpu-baseline --no-e2e > gpurun_out/r2t_${cfg}_$name.json 2> gpurun_out/r2t_${cfg}_$name.err
  done
}
B1=SSPD_LIB=$PWD/variants/libsspd_cuda_bw1.so
B8=SSPD_LIB=$PWD/variants/libsspd_cuda_bw8.so
run pairset SSPD_CSET=0
run bw4_25 SSPD_CSET_LOG2=25
run bw4_25h SSPD_CSET_LOG2=25 SSPD_DEDUP_PIPE=1
run bw4_24h SSPD_CSET_LOG2=24 SSPD_DEDUP_PIPE=1
run bw4_26h SSPD_CSET_LOG2=26 SSPD_DEDUP_PIPE=1
run bw8_25h $B8 SSPD_CSET_LOG2=25 SSPD_DEDUP_PIPE=1
run bw8_24h $B8 SSPD_CSET_LOG2=24 SSPD_DEDUP_PIPE=1
run bw1_25h $B1 SSPD_CSET_LOG2=25 SSPD_DEDUP_PIPE=1
run pairset_b SSPD_CSET=0
