# Round-2 A/B: the pipelined scan LOADS (ld.cg) each fresh pair's recorders when it hashes them, so the
# deferred atomics hit L2 (-DSSPD_PIPE_LDPF=1 values unused / 2 carried), variants q..u in variants/.
#   /usr/local/graft/bin/gpurun --timeout 2400 -- 'bash tools/r02_ab_ldpf.sh'
mkdir -p gpurun_out
for cfg in c2 c2p64; do
  python bench.py --config $cfg --no-cpu-baseline --no-e2e > gpurun_out/r2l_${cfg}_a.json 2> gpurun_out/r2l_${cfg}_a.err
  for n in q r s t u; do
    SSPD_LIB=$PWD/variants/libsspd_cuda_$n.so python bench.py --config $cfg --no-cpu-baseline --no-e2e > gpurun_out/r2l_${cfg}_$n.json 2> gpurun_out/r2l_${cfg}_$n.err
  done
done
