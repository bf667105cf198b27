cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
for v in "" "hot_window=-1" "scatter_stripes=32" "scatter_run=8" "scatter_run=1" "l2_persist=-1"; do
  echo "== $v"; timeout 300 python scripts/exp_passfit.py C4 -1 $v 2>&1 | grep -E "fit|totals|^C4"
done > gpurun_out/passfit_var.log
cat gpurun_out/passfit_var.log
