# round-2 near-edge pull: GPU tests + C4/C2 A/B
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pull.py -x -q > gpurun_out/pull_tests.log 2>&1; echo "pull tests rc=$?"
tail -5 gpurun_out/pull_tests.log
DITER_TRACE=1 timeout 900 python scripts/exp_pull.py C4 "-1:0 1:0 1:60 1:200 1:1" 5 > gpurun_out/pull_ab_c4.log 2> gpurun_out/pull_ab_c4.err; echo "ab rc=$?"
cat gpurun_out/pull_ab_c4.log; grep "pull" gpurun_out/pull_ab_c4.err | head -20
