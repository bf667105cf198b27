# 32-bit col_ptr copy in the sweep scan: sweep tests, dist sweep tests, A/B timing on C4 / C3
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_sweep.py tests/test_gpu_dist.py -q -k "sweep or pilot or sleep" > gpurun_out/r4_cp32_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r4_cp32_tests.log
for c in C4 C3; do
  echo "$c $(timeout 600 python scripts/sweep.py --config $c --reps 4 --variants "sweep=1,scatter_stripes=$([ $c = C4 ] && echo 4 || echo 8),scatter_run=$([ $c = C4 ] && echo 6 || echo 1)" 2>&1 | tail -1)"
done 2>&1 | tee gpurun_out/r4_cp32.txt
