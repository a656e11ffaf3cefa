# Round-2 A/B #14 (rejected; the kernel change is profiles/r02_ab_ringv4.patch -- apply it first): the window ring cell-major in f32 counts (-DSSPD_RING_V4=1), so a recorder's move
# (+1 into now's slot, -1 out of its old one) is one red.global.add.v4.f32 when both slots share a
# 16 B group, against the default slot-major u32 ring (two reds per move).  Variants:
#   nvcc <the Makefile's NVFLAGS> -DSSPD_RING_V4=1 [-DSSPD_CHECKED] -shared -o variants/libsspd_cuda_v4[_checked].so paper_1803_11036_b200/csrc/sspd_cuda.cu -lgomp
#   /usr/local/graft/bin/gpurun --timeout 3000 -- 'bash tools/r02_ab_ringv4.sh'
mkdir -p gpurun_out
T=${TAG:-r4l}
S="tests/test_gpu_parity.py tests/test_gpu_narrow.py tests/test_gpu_fuzz.py tests/test_gpu_keyset.py"
SSPD_LIB=$PWD/variants/libsspd_cuda_v4.so timeout 1500 python -m pytest -q -m "gpu and not slow" -p no:cacheprovider $S > gpurun_out/${T}_pytest_v4.log 2>&1
tail -1 gpurun_out/${T}_pytest_v4.log
SSPD_LIB=$PWD/variants/libsspd_cuda_v4_checked.so SSPD_CHECKED_ASSERT=1 timeout 1500 python -m pytest -q -m "gpu and not slow" -p no:cacheprovider $S > gpurun_out/${T}_pytest_v4_checked.log 2>&1
tail -1 gpurun_out/${T}_pytest_v4_checked.log
run() {  # name, env...
  local name=$1; shift
  for cfg in c2 c2p64 c1; do
    timeout 600 env "$@" python bench.py --config $cfg --no-cpu-baseline --no-e2e > gpurun_out/${T}_${cfg}_$name.json 2> gpurun_out/${T}_${cfg}_$name.err
  done
}
run base
run v4 SSPD_LIB=$PWD/variants/libsspd_cuda_v4.so
run base_b
run v4_b SSPD_LIB=$PWD/variants/libsspd_cuda_v4.so
