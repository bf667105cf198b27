cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/test_gpu_dist.py tests/test_gpu_ipc.py -v --timeout 900 -k "p2p" > gpurun_out/gpu_p2p.log 2>&1; echo p2p_rc=$?
grep -E "PASS|FAIL|Error|error|assert" gpurun_out/gpu_p2p.log | head -30
