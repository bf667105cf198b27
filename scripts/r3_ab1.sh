# A/B: H by plain load+store, hot-window sizes (k_sweep, bench launch configuration)
cd ${GRAFT_REPO_ROOT:-.}
run() { c=$1; v=$2
  if [ $v = base ]; then L=""; else L="DITER_LIB=$PWD/variants/v_$v.so"; fi
  echo "$c $v $(env $L timeout 600 python scripts/sweep.py --config $c --reps 4 --variants "sweep=1,scatter_stripes=$([ $c = C4 ] && echo 4 || echo 8),scatter_run=$([ $c = C4 ] && echo 6 || echo 1)" 2>&1 | tail -1)"
}
for v in base hplain hplain2 hot256 hot512 hot1024 base; do run C4 $v; done
for v in base hplain hplain2 hot512; do run C3 $v; done
