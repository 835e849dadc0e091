timeout 900 python -m pytest tests/test_gpu_scores_codes.py -q -x -p no:cacheprovider > gpurun_out/pytest_sc.log 2>&1; tail -25 gpurun_out/pytest_sc.log
