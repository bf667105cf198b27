cd ${GRAFT_REPO_ROOT:-.}
timeout 900 python scripts/sweep.py --config C4 --reps 3 --variants "sweep=1,scatter_stripes=4,scatter_run=6,l2_persist=24;sweep=1,scatter_stripes=4,scatter_run=6,l2_persist=28;sweep=1,scatter_stripes=4,scatter_run=6,l2_persist=32;sweep=1,scatter_stripes=4,scatter_run=6,l2_persist=36;sweep=1,scatter_stripes=4,scatter_run=6,l2_persist=20" 2>&1
timeout 900 python scripts/sweep.py --config C3 --reps 3 --variants "sweep=1,scatter_run=1,l2_persist=32;sweep=1,scatter_run=1,l2_persist=36;sweep=1,scatter_run=1,l2_persist=44;sweep=1,scatter_run=1,l2_persist=48" 2>&1
