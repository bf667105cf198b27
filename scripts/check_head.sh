# Full -m gpu suite + smoke + default bench line on the current tree (one B200)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q --timeout 1200 > gpurun_out/gpu_tests_all.log 2>&1; echo tests_rc=$?; tail -4 gpurun_out/gpu_tests_all.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo c4_rc=$?; tail -c 600 gpurun_out/bench_c4.json
