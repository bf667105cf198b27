# Re-entry validation of HEAD: smoke, every -m gpu test (full scale included), default bench lines
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r3_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r3_smoke.log
timeout 3000 python -m pytest tests -m gpu -x -q --timeout 1500 > gpurun_out/r3_gpu_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r3_gpu_tests.log
python bench.py > gpurun_out/r3_bench_c4.json 2> gpurun_out/r3_bench_c4.err; echo "c4 rc=$?"; cat gpurun_out/r3_bench_c4.json
python bench.py --config C3 --steps 10 --warmup 3 > gpurun_out/r3_bench_c3.json 2>/dev/null; echo "c3 rc=$?"; cat gpurun_out/r3_bench_c3.json
