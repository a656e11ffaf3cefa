./tools/bin/bench_api > gpurun_out/bench_api.md 2>&1
