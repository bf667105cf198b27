cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
V="sweep=1;sweep=1,scatter_stripes=4;sweep=1,scatter_stripes=16;sweep=1,scatter_stripes=32;sweep=1,scatter_stripes=1;sweep=1,hybrid_frac=0.7;sweep=1,hybrid_frac=0.4;sweep=1,alpha=1.8;sweep=1,alpha=1.5;sweep=1,select_key=2;sweep=1,policy=0"
timeout 1200 python scripts/sweep.py --config C4 --reps 2 --variants "$V" > gpurun_out/sweep_tune_c4.log 2>&1
cat gpurun_out/sweep_tune_c4.log
for c in C3 C2 C5; do timeout 600 python scripts/sweep.py --config $c --reps 3 --variants "sweep=0;sweep=1;sweep=1,scatter_run=1;sweep=1,scatter_stripes=16" 2>&1; done > gpurun_out/sweep_tune_other.log
cat gpurun_out/sweep_tune_other.log
