cd ${GRAFT_REPO_ROOT:-.}
timeout 900 python -m pytest tests/test_gpu_sweep.py -x -q --timeout 600 2>&1 | tail -8
DITER_LIB=$PWD/variants/v_win2.so timeout 900 python -m pytest tests/test_gpu_sweep.py -x -q --timeout 600 -k "win or web" 2>&1 | tail -4
run() { c=$1; v=$2; opts=$3
  if [ $v = base ]; then L=""; else L="DITER_LIB=$PWD/variants/v_$v.so"; fi
  echo "$c $v $(env $L timeout 600 python scripts/sweep.py --config $c --reps 3 --variants "$opts" 2>&1 | tail -1)"
}
run C4 base "sweep=1,scatter_stripes=4,scatter_run=6"
for r in 8 16 32; do run C4 base "sweep=2,scatter_run=$r"; done
for r in 8 16 32 64; do run C4 win2 "sweep=2,scatter_run=$r"; done
run C3 base "sweep=2,scatter_run=16"
run C3 win2 "sweep=2,scatter_run=16"
