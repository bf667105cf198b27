cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_dist.py -v -x --timeout 700 -k "async_parity" > gpurun_out/gpu_dist.log 2>&1; echo dist_rc=$?; grep -E "PASS|FAIL|Error|error" gpurun_out/gpu_dist.log | head -20
timeout 300 python scripts/profile_run.py --config C4 --max-passes 10 > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_scatter" -s 6 -c 2 -o gpurun_out/r02_scatter_pipe python scripts/profile_run.py --config C4 --max-passes 10 > gpurun_out/ncu_full.log 2>&1
echo full_rc=$?
