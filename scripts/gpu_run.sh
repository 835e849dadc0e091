timeout 300 python -m pytest tests/test_gpu_scores_codes.py -x -q 2>&1 | tail -8
