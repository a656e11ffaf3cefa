python -m pytest tests/test_gpu_parity.py -q -x -k "input_forms" > gpurun_out/pytest_forms.log 2>&1
