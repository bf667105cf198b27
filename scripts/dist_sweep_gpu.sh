cd ${GRAFT_REPO_ROOT:-.}
timeout 1500 python -m pytest tests/test_gpu_dist.py -x -q -k "sweeps_on_ranks or p2p_parity or async_parity" 2>&1 | tail -15
