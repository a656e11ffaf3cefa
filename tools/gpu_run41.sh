python -m pytest tests/test_cpp_api.py tests/test_cli.py -q -m gpu > gpurun_out/pytest_cpp.log 2>&1
