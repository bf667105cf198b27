# Final tree with options.key_offset (C4 c = 8, f = 0.55): tests of the changed paths, bench lines, launch list, traffic, full-scale parity
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_sweep.py tests/test_gpu_bench_contract.py -q > gpurun_out/r02g_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r02g_tests.log
python bench.py --steps 20 --warmup 5 > gpurun_out/r02g_bench_c4.json 2> gpurun_out/r02g_bench_c4.err; echo "c4 rc=$?"
python bench.py --config C3 --steps 10 --warmup 3 > gpurun_out/r02g_bench_c3.json 2>/dev/null; echo "C3 rc=$?"
python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/r02g_bench_c4_reference.json 2>/dev/null; echo "ref rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r02g_launches_c4.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-raw-key --no-snapshot > /dev/null 2>&1; echo "launches c4 rc=$?"
cp profiles/ncu_traffic.json gpurun_out/ncu_traffic.json
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum -k regex:k_sweep --clock-control none --csv \
  --log-file gpurun_out/r02g_traffic_C4.csv python scripts/profile_run.py --config C4 --max-passes 1000 --pass-csv gpurun_out/r02g_passes_C4.csv > /dev/null 2>&1
python scripts/ncu_traffic.py --config C4 --kernel k_sweep --n 100000000 --launches gpurun_out/r02g_traffic_C4.csv --passes gpurun_out/r02g_passes_C4.csv --out gpurun_out/ncu_traffic.json | grep traffic_over
timeout 1500 python -m pytest tests/test_gpu_full_scale.py -q -s -k "c4_full" 2>&1 | grep -E "C4:|C3:|passed|failed" > gpurun_out/r02g_full_scale_parity.txt; cat gpurun_out/r02g_full_scale_parity.txt
