timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "fp32" > gpurun_out/pytest_fp32.log 2>&1; echo fp32=$?; tail -25 gpurun_out/pytest_fp32.log
