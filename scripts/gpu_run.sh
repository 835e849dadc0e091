timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_lowbit.py tests/test_gpu_append.py -q -x 2>&1 | tail -3
