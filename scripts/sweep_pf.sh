cd ${GRAFT_REPO_ROOT:-.}
timeout 900 python -m pytest tests/test_gpu_sweep.py -x -q 2>&1 | tail -2
timeout 900 python scripts/sweep.py --config C4 --reps 3 --variants "sweep=1,scatter_stripes=4;sweep=1,scatter_stripes=4,scatter_run=4;sweep=1,scatter_stripes=4,scatter_run=6;sweep=1,scatter_stripes=4,scatter_run=2" 2>&1
timeout 900 python scripts/sweep.py --config C3 --reps 3 --variants "sweep=1;sweep=1,scatter_run=2;sweep=1,scatter_run=3" 2>&1
