python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1
python -c "import __graft_entry__ as G; G.smoke()" > gpurun_out/smoke.log 2>&1
python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
