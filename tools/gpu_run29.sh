python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1
python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1
python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
python bench.py --config c1 > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
