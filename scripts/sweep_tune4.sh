cd ${GRAFT_REPO_ROOT:-.}
V="sweep=1,scatter_stripes=4,scatter_run=6;sweep=1,scatter_stripes=4,scatter_run=6,hybrid_frac=0.5;sweep=1,scatter_stripes=4,scatter_run=6,hybrid_frac=0.7;sweep=1,scatter_stripes=4,scatter_run=8;sweep=1,scatter_stripes=2,scatter_run=6;sweep=1,scatter_stripes=4,scatter_run=6,alpha=1.8"
timeout 1200 python scripts/sweep.py --config C4 --reps 3 --variants "$V" 2>&1
V="sweep=1,scatter_run=1;sweep=1,scatter_run=1,hybrid_frac=0.6;sweep=1,scatter_run=1,hybrid_frac=0.7;sweep=1,scatter_run=4;sweep=1,scatter_run=1,scatter_stripes=16"
timeout 1200 python scripts/sweep.py --config C3 --reps 3 --variants "$V" 2>&1
