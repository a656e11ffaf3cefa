# Round-2 A/B #13 of the key-set scan (rejected; the kernel change is profiles/r02_ab_deep.patch -- apply it first): old stamps consumed two iterations after their atomics
# (-DSSPD_CSET_DEEP=1, the body alternating between two old-value arrays) at 4 / 3 / 2 CTAs per SM
# (-DSSPD_PIPE_MINB), against the default (one iteration).  Variants:
#   nvcc <the Makefile's NVFLAGS> -DSSPD_CSET_DEEP=1 [-DSSPD_PIPE_MINB=3|2] -shared -o variants/libsspd_cuda_deep{4,3,2}.so paper_1803_11036_b200/csrc/sspd_cuda.cu -lgomp
#   /usr/local/graft/bin/gpurun --timeout 2400 -- 'bash tools/r02_ab_deep.sh'
mkdir -p gpurun_out
T=${TAG:-r4k}
SSPD_LIB=$PWD/variants/libsspd_cuda_deep3.so timeout 900 python -m pytest tests/test_gpu_keyset.py -q -x -k "bit_exact or distinct" > gpurun_out/${T}_pytest_deep3.log 2>&1
tail -1 gpurun_out/${T}_pytest_deep3.log
run() {  # name, env...
  local name=$1; shift
  for cfg in c2 c2p64; do
    timeout 600 env "$@" python bench.py --config $cfg --no-cpu-baseline --no-e2e > gpurun_out/${T}_${cfg}_$name.json 2> gpurun_out/${T}_${cfg}_$name.err
  done
}
run base
run deep4 SSPD_LIB=$PWD/variants/libsspd_cuda_deep4.so
run deep3 SSPD_LIB=$PWD/variants/libsspd_cuda_deep3.so
run deep2 SSPD_LIB=$PWD/variants/libsspd_cuda_deep2.so
run base_b
