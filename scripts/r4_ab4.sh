# A/B: derived per-edge key |F_i| / (#out_i + c)
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
run() { c=$1; v=$2; extra=$3
  if [ $v = base ]; then L=""; else L="DITER_LIB=$PWD/variants/v_$v.so"; fi
  echo "$c $v $extra $(env $L timeout 600 python scripts/sweep.py --config $c --reps 3 --variants "sweep=1,scatter_stripes=$([ $c = C4 ] && echo 4 || echo 8),scatter_run=$([ $c = C4 ] && echo 6 || echo 1)$extra" 2>&1 | tail -1)"
}
for v in base ko0.5 ko2.0 ko4.0 ko8.0; do run C4 $v ""; done 2>&1 | tee gpurun_out/r4_ab4.txt
for v in ko2.0 ko4.0; do for f in 0.5 0.7; do run C4 $v ",hybrid_frac=$f"; done; done 2>&1 | tee -a gpurun_out/r4_ab4.txt
for v in base ko2.0 ko4.0; do run C3 $v ""; done 2>&1 | tee -a gpurun_out/r4_ab4.txt
