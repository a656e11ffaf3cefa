# Round-end style verification on a B200 (run through gpurun from the repo root):
#   /usr/local/graft/bin/gpurun --timeout 2400 -- 'bash tools/gpu_verify.sh'
# GPU tests, smoke, the default bench line (C2) with the CPU reference beside it, C1, and the
# reference arm.  Outputs land in gpurun_out/.
python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1
python -c "import __graft_entry__ as G; G.smoke()" > gpurun_out/smoke.log 2>&1
python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
python bench.py --config c1 > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
./tools/bin/bench_api > gpurun_out/bench_api.md 2>&1
