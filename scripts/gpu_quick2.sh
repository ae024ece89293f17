cd $GRAFT_REPO_ROOT
python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_kb.py tests/test_gpu_direct.py -q -k "edge or fuzz or 1e-12 or confined or c1_" 2>&1 | tail -6
