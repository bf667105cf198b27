# Round-2 session 5: A/B of L2 evict-first hints on the sweep's streaming data, trimmed edge slots, lower hub limit
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
run() { c=$1; v=$2
  if [ $v = base ]; then L=""; else L="DITER_LIB=$PWD/variants/v_$v.so"; fi
  echo "$c $v $(env $L timeout 600 python scripts/sweep.py --config $c --reps 4 --variants "sweep=1,scatter_stripes=$([ $c = C4 ] && echo 4 || echo 8),scatter_run=$([ $c = C4 ] && echo 6 || echo 1)" 2>&1 | tail -1)"
}
for v in base ef1 ef2 ef3 ef7 trim trim_fold base; do run C4 $v; done 2>&1 | tee gpurun_out/r4_ab2.txt
for v in base ef1 ef3 ef7 trim mid2048 mid4096; do run C3 $v; done 2>&1 | tee -a gpurun_out/r4_ab2.txt
