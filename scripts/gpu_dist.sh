timeout 900 python -m pytest tests/test_dist_gpu.py -q -x > gpurun_out/pytest_dist.log 2>&1; echo dist=$?; tail -30 gpurun_out/pytest_dist.log
