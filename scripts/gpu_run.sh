timeout 900 python -m pytest tests/test_gpu_fp8.py -q -x -p no:cacheprovider > gpurun_out/pytest_fp8.log 2>&1; tail -25 gpurun_out/pytest_fp8.log
