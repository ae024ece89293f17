cd $GRAFT_REPO_ROOT
python -m pytest tests/test_gpu_parity.py -q -x -k "general_b or c1_ or edge" --durations=3 2>&1 | tail -5
