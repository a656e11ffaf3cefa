for pl in 0 1; do
  echo "== w16 preload $pl" >> gpurun_out/ab_narrow_preload.txt
  SSPD_NARROW_PRELOAD=$pl python bench.py --stamp-width 16 --steps 10 --no-cpu-baseline --no-e2e >> gpurun_out/ab_narrow_preload.txt 2>&1
done
SSPD_NARROW_PRELOAD=1 python -m pytest tests/test_gpu_narrow.py -q -x -k "width16 or equals_wide" > gpurun_out/pytest_narrow_pl.log 2>&1
