# Round-2 A/B #2 of the compact key set: the 3-round 48-bit permutation vs one multiply
# (variants/libsspd_cuda_p1.so, -DSSPD_CSET_PERM=1), at 2^25 entries, with and without L2 priorities.
#   /usr/local/graft/bin/gpurun --timeout 3000 -- 'bash tools/r02_ab_cset2.sh'
mkdir -p gpurun_out
python -m pytest tests/test_gpu_keyset.py -q > gpurun_out/r2s_pytest_keyset.log 2>&1
SSPD_LIB=$PWD/variants/libsspd_cuda_p1.so python -m pytest tests/test_gpu_keyset.py -q > gpurun_out/r2s_pytest_keyset_p1.log 2>&1
run() {  # name, env...
  local name=$1; shift
  for cfg in c2 c2p64; do
    env "$@" python bench.py --config $cfg --no-cpu-baseline --no-e2e > gpurun_out/r2s_${cfg}_$name.json 2> gpurun_out/r2s_${cfg}_$name.err
  done
}
P1=SSPD_LIB=$PWD/variants/libsspd_cuda_p1.so
run pairset SSPD_CSET=0
run cset25 SSPD_CSET_LOG2=25
run cset25h SSPD_CSET_LOG2=25 SSPD_DEDUP_PIPE=1
run p1_25 $P1 SSPD_CSET_LOG2=25
run p1_25h $P1 SSPD_CSET_LOG2=25 SSPD_DEDUP_PIPE=1
run p1_26h $P1 SSPD_CSET_LOG2=26 SSPD_DEDUP_PIPE=1
run pairset_b SSPD_CSET=0
run cset25h_b SSPD_CSET_LOG2=25 SSPD_DEDUP_PIPE=1
