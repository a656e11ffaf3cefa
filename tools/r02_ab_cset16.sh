# Round-2 A/B #16: 16-bit grids' dedup scan on the pipelined key-set kernel (scan_cset_kernel on bf16
# codes) against the narrow pair-set scan ($SSPD_CSET=0).  Parity first (narrow, fuzz, key-set suites and
# the checked build's suites), then the C4 sweep at w = 16 and a C2 sanity line at w = 32.
#   /usr/local/graft/bin/gpurun --timeout 3000 -- 'bash tools/r02_ab_cset16.sh'
mkdir -p gpurun_out
T=${TAG:-r4p}
timeout 1500 python -m pytest -q tests/test_gpu_narrow.py tests/test_gpu_fuzz.py tests/test_gpu_keyset.py > gpurun_out/${T}_pytest.log 2>&1
tail -1 gpurun_out/${T}_pytest.log
timeout 1500 python -m pytest -q tests/test_gpu_checked.py > gpurun_out/${T}_pytest_checked.log 2>&1
tail -1 gpurun_out/${T}_pytest_checked.log
timeout 900 python tools/sweep_c4.py --widths 16 --out gpurun_out/${T}_c4_w16.md > gpurun_out/${T}_c4.log 2>&1
SSPD_CSET=0 timeout 900 python tools/sweep_c4.py --widths 16 --out gpurun_out/${T}_c4_w16_pairset.md > gpurun_out/${T}_c4p.log 2>&1
tail -7 gpurun_out/${T}_c4_w16.md; tail -7 gpurun_out/${T}_c4_w16_pairset.md
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/${T}_c2.json 2> gpurun_out/${T}_c2.err
