# A/B: hub-kernel grid (occupancy vs 3 CTAs/SM) on C3; the paper key under sweeps on C4/C3
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
for r in 1 2; do for v in base h3; do
  if [ $v = base ]; then L=""; else L="DITER_LIB=$PWD/variants/v_$v.so"; fi
  echo "C3 $v $(env $L timeout 300 python scripts/sweep.py --config C3 --reps 3 --variants "sweep=1,scatter_stripes=8,scatter_run=1;sweep=0,hybrid_frac=0.05,scatter_run=1" 2>&1 | tr '\n' ' ')"
done; done
V="sweep=1,scatter_stripes=4,scatter_run=6;sweep=1,scatter_stripes=4,scatter_run=6,select_key=2;sweep=1,scatter_stripes=4,scatter_run=6,select_key=2,hybrid_frac=0.4;sweep=1,scatter_stripes=4,scatter_run=6,select_key=2,hybrid_frac=0.75;sweep=1,scatter_stripes=4,scatter_run=6,select_key=2,alpha=1.6"
timeout 900 python scripts/sweep.py --config C4 --reps 3 --variants "$V" 2>&1
