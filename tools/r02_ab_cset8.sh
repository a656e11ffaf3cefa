# Round-2 A/B #17: 8-bit grids' dedup scan on the pipelined key-set kernel ($SSPD_CSET8=1: each touch a
# load and a CAS on the containing word) against the unpipelined pair-set narrow scan (default).
#   /usr/local/graft/bin/gpurun --timeout 2400 -- 'bash tools/r02_ab_cset8.sh'
mkdir -p gpurun_out
T=${TAG:-r4r}
SSPD_CSET8=1 timeout 900 python -m pytest -q tests/test_gpu_narrow.py tests/test_gpu_fuzz.py -k "width8 or fuzz" > gpurun_out/${T}_pytest_cset8.log 2>&1
tail -1 gpurun_out/${T}_pytest_cset8.log
SSPD_CSET8=1 timeout 900 python tools/sweep_c4.py --widths 8 --out gpurun_out/${T}_c4_w8_cset.md > gpurun_out/${T}_c4.log 2>&1
tail -6 gpurun_out/${T}_c4_w8_cset.md
