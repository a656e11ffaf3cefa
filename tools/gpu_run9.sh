python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1
python tools/sweep_c4.py --out gpurun_out/c4.md > gpurun_out/c4.log 2>&1
python tools/sweep_c5.py --out gpurun_out/c5.md > gpurun_out/c5.log 2>&1
python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
python bench.py --config c1 > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
echo done
