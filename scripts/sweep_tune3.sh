cd ${GRAFT_REPO_ROOT:-.}
V="sweep=1,hybrid_frac=0.6;sweep=1,hybrid_frac=0.6,scatter_stripes=4;sweep=1,hybrid_frac=0.55;sweep=1,hybrid_frac=0.65;sweep=1,hybrid_frac=0.6,alpha=1.8;sweep=1,hybrid_frac=0.6,scatter_stripes=6"
timeout 1200 python scripts/sweep.py --config C4 --reps 3 --variants "$V" 2>&1
V="sweep=1,hybrid_frac=0.3;sweep=1,hybrid_frac=0.4;sweep=1,hybrid_frac=0.5;sweep=1,hybrid_frac=0.3,scatter_run=2;sweep=1,hybrid_frac=0.3,select_key=2;sweep=1,hybrid_frac=0.3,alpha=1.3"
timeout 1200 python scripts/sweep.py --config C3 --reps 3 --variants "$V" 2>&1
