python tools/sweep_c4.py --config c2 --widths 8,16,32 --out gpurun_out/c4_sweep.md > gpurun_out/c4_sweep.log 2>&1
