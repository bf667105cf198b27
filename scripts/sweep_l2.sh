cd ${GRAFT_REPO_ROOT:-.}
timeout 900 python scripts/sweep.py --config C4 --reps 3 --variants "sweep=1,scatter_stripes=4,scatter_run=6;sweep=1,scatter_stripes=4,scatter_run=6,l2_persist=-1;sweep=1,scatter_stripes=4,scatter_run=6,l2_persist=12;sweep=1,scatter_stripes=4,scatter_run=6,l2_persist=28;sweep=1,scatter_stripes=4,scatter_run=6,l2_persist=40" 2>&1
timeout 900 python scripts/sweep.py --config C3 --reps 3 --variants "sweep=1,scatter_run=1;sweep=1,scatter_run=1,l2_persist=-1;sweep=1,scatter_run=1,l2_persist=16;sweep=1,scatter_run=1,l2_persist=40;sweep=1,scatter_run=1,l2_persist=56" 2>&1
