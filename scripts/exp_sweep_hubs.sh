# In-kernel hub chunks under sweeps: GPU tests, then A/B against the two-kernel build
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sweep.py -x -q --timeout 600 2>&1 | tail -5
timeout 900 python -m pytest tests/test_gpu_dist.py -x -q --timeout 600 -k "sweep" 2>&1 | tail -3
for r in 1 2; do for v in base nohub cas; do
  if [ $v = base ]; then L=""; else L="DITER_LIB=$PWD/variants/v_$v.so"; fi
  echo "C3 $v $(env $L timeout 300 python scripts/sweep.py --config C3 --reps 3 --variants "sweep=1,scatter_stripes=8,scatter_run=1" 2>&1 | tr '\n' ' ')"
  echo "C4 $v $(env $L timeout 300 python scripts/sweep.py --config C4 --reps 3 --variants "sweep=1,scatter_stripes=4,scatter_run=6" 2>&1 | tr '\n' ' ')"
done; done
