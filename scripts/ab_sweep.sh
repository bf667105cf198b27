# A/B of k_sweep builds (variants/) on C4 / C3 in the bench launch configuration
cd ${GRAFT_REPO_ROOT:-.}
for c in C4 C3; do for r in 1 2; do for v in base kw; do
  if [ $v = base ]; then L=""; else L="DITER_LIB=$PWD/variants/v_$v.so"; fi
  echo "$c $v $(env $L timeout 300 python scripts/sweep.py --config $c --reps 3 --variants "sweep=1,scatter_stripes=$([ $c = C4 ] && echo 4 || echo 8),scatter_run=$([ $c = C4 ] && echo 6 || echo 1)" 2>&1 | tail -1)"
done; done; done
