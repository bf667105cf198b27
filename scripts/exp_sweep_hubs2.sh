# In-kernel hub chunks: mid-sweep polling variant (tests + C3 A/B)
cd ${GRAFT_REPO_ROOT:-.}
DITER_LIB=$PWD/variants/v_poll.so timeout 900 python -m pytest tests/test_gpu_sweep.py -x -q --timeout 600 -k "hub" 2>&1 | tail -2
for r in 1 2; do for v in base poll; do
  if [ $v = base ]; then L=""; else L="DITER_LIB=$PWD/variants/v_$v.so"; fi
  echo "C3 $v $(env $L timeout 300 python scripts/sweep.py --config C3 --reps 3 --variants "sweep=1,scatter_stripes=8,scatter_run=1;sweep=1,scatter_stripes=8,scatter_run=2" 2>&1 | tr '\n' ' ')"
done; done
