cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_bench_contract.py -v --timeout 900 > gpurun_out/bench_contract.log 2>&1; echo contract_rc=$?
grep -E "PASS|FAIL|Error|assert" gpurun_out/bench_contract.log | head -20
timeout 600 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?; tail -2 gpurun_out/smoke.log
