cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_sweep.py -x -q 2>&1 | tail -2
timeout 600 python scripts/sweep.py --config C5 --reps 3 --variants "sweep=0;sweep=1" 2>&1
V="sweep=1,hybrid_frac=0.7;sweep=1,hybrid_frac=0.7,alpha=1.8;sweep=1,hybrid_frac=0.7,scatter_stripes=4;sweep=1,hybrid_frac=0.8;sweep=1,hybrid_frac=0.9;sweep=1,hybrid_frac=0.7,scatter_run=2;sweep=1,hybrid_frac=0.7,scatter_run=4;sweep=1,hybrid_frac=0.6"
timeout 1200 python scripts/sweep.py --config C4 --reps 2 --variants "$V" 2>&1
V="sweep=1;sweep=1,hybrid_frac=0.1;sweep=1,hybrid_frac=0.2;sweep=1,hybrid_frac=0.3;sweep=1,alpha=2.0;sweep=1,alpha=2.0,hybrid_frac=0.2;sweep=1,scatter_stripes=4"
timeout 1200 python scripts/sweep.py --config C3 --reps 2 --variants "$V" 2>&1
