# Round-2 final measurements of the sweep launch configuration (profiles/r02s_*)
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
python bench.py --steps 20 --warmup 5 > gpurun_out/r02s_bench_c4.json 2> gpurun_out/r02s_bench_c4.err; echo "c4 rc=$?"
for c in C3 C2 C5 C1; do python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/r02s_bench_$(echo $c | tr C c).json 2>/dev/null; echo "$c rc=$?"; done
python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/r02s_bench_c4_reference.json 2>/dev/null; echo "ref rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r02s_launches_c4.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-raw-key --no-snapshot > /dev/null 2>&1; echo "launches c4 rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r02s_launches_c3.csv \
  python bench.py --config C3 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-snapshot > /dev/null 2>&1; echo "launches c3 rc=$?"
cp profiles/ncu_traffic.json gpurun_out/ncu_traffic.json
for c in C4 C3; do
  n=100000000; [ $c = C3 ] && n=16777216
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum -k regex:k_sweep --clock-control none --csv \
    --log-file gpurun_out/r02s_traffic_$c.csv python scripts/profile_run.py --config $c --max-passes 1000 --pass-csv gpurun_out/r02s_passes_$c.csv > /dev/null 2>&1
  python scripts/ncu_traffic.py --config $c --kernel k_sweep --n $n --launches gpurun_out/r02s_traffic_$c.csv --passes gpurun_out/r02s_passes_$c.csv --out gpurun_out/ncu_traffic.json | grep traffic_over
done
ncu --set full --clock-control none --import-source on -k regex:k_sweep --launch-skip 4 --launch-count 2 -o gpurun_out/r02s_sweep_c4 -f \
  python scripts/profile_run.py --config C4 --max-passes 8 > /dev/null 2>&1; echo "full c4 rc=$?"
timeout 1500 python -m pytest tests/test_gpu_full_scale.py -q -s -k "c4_full or c3_full" 2>&1 | grep -E "C4:|C3:|passed|failed" > gpurun_out/r02s_full_scale_parity.txt; cat gpurun_out/r02s_full_scale_parity.txt
