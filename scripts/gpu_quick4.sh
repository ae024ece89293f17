cd $GRAFT_REPO_ROOT
python -m pytest tests/test_gpu_parity.py tests/test_gpu_direct.py tests/test_gpu_kb.py -q -k "s1 or confined or edge or c1_ or direct_c" --durations=5 2>&1 | tail -9
