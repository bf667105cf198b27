cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_sweep.py -x -q > gpurun_out/sweep_tests.log 2>&1; echo "sweep tests rc=$?"
tail -15 gpurun_out/sweep_tests.log
timeout 900 python scripts/sweep.py --config C4 --reps 3 --variants "sweep=0;sweep=1;sweep=1,scatter_run=1;sweep=1,scatter_run=4;sweep=1,hybrid_frac=0.3;sweep=1,select_key=0,hybrid_frac=0.15" > gpurun_out/sweep_ab_c4.log 2>&1; echo "ab rc=$?"
cat gpurun_out/sweep_ab_c4.log
