# Schedule grid for C4 sweeps: alpha x hybrid_frac (+ the paper key)
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
V=""
for a in 2.0 3.0 4.0; do for f in 0.5 0.6 0.7; do V="$V;sweep=1,scatter_stripes=4,scatter_run=6,alpha=$a,hybrid_frac=$f"; done; done
V="$V;sweep=1,scatter_stripes=4,scatter_run=6,select_key=2;sweep=1,scatter_stripes=4,scatter_run=6,alpha=1.5,hybrid_frac=0.6;sweep=1,scatter_stripes=4,scatter_run=6,alpha=8.0,hybrid_frac=0.6"
timeout 1500 python scripts/sweep.py --config C4 --reps 3 --variants "${V#;}" 2>&1 | grep "ms=" | tee gpurun_out/r4_sched_c4.txt
V=""
for a in 1.5 2.0 3.0; do for f in 0.4 0.5 0.6; do V="$V;sweep=1,scatter_stripes=8,scatter_run=1,alpha=$a,hybrid_frac=$f"; done; done
timeout 1500 python scripts/sweep.py --config C3 --reps 3 --variants "${V#;}" 2>&1 | grep "ms=" | tee gpurun_out/r4_sched_c3.txt
