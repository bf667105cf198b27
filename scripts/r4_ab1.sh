# Round-2 session 5: A/B of k_sweep build variants (bench launch configuration) + source-level ncu of the base
# (variants/ built with scripts/build_variant.py; the rowpf flag, DITER_SWEEP_ROW_PF, was removed again after this run)
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
run() { c=$1; v=$2
  if [ $v = base ]; then L=""; else L="DITER_LIB=$PWD/variants/v_$v.so"; fi
  echo "$c $v $(env $L timeout 600 python scripts/sweep.py --config $c --reps 4 --variants "sweep=1,scatter_stripes=$([ $c = C4 ] && echo 4 || echo 8),scatter_run=$([ $c = C4 ] && echo 6 || echo 1)" 2>&1 | tail -1)"
}
for v in base fold rowpf1 rowpf2 un5 un8 occ4 takered base; do run C4 $v; done 2>&1 | tee gpurun_out/r4_ab1.txt
for v in base fold un5 occ4; do run C3 $v; done 2>&1 | tee -a gpurun_out/r4_ab1.txt
ncu --set full --clock-control none --import-source on -k regex:k_sweep --launch-skip 9 --launch-count 1 -o gpurun_out/r4_sweep_c4_dense -f \
  python scripts/profile_run.py --config C4 --max-passes 12 > gpurun_out/ncu_r4_dense.log 2>&1; echo "dense rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_sweep --launch-skip 40 --launch-count 1 -o gpurun_out/r4_sweep_c4_late -f \
  python scripts/profile_run.py --config C4 --max-passes 44 > gpurun_out/ncu_r4_late.log 2>&1; echo "late rc=$?"
ls -la gpurun_out/*.ncu-rep
