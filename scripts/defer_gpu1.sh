# far-edge deferral: GPU tests + C4 A/B
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_defer.py -x -q > gpurun_out/defer_tests.log 2>&1; echo "defer tests rc=$?"
tail -15 gpurun_out/defer_tests.log
timeout 900 python scripts/exp_defer.py C4 "-1:0 2:0 4:0 8:0 16:0" 5 > gpurun_out/defer_ab_c4.log 2>&1; echo "ab rc=$?"
cat gpurun_out/defer_ab_c4.log
