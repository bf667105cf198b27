# Final tree (32-bit col_ptr copy in the sweep scan): bench lines C4 / C3, launch lists, per-launch traffic
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
python bench.py --steps 20 --warmup 5 > gpurun_out/r02h_bench_c4.json 2> gpurun_out/r02h_bench_c4.err; echo "c4 rc=$?"
python bench.py --config C3 --steps 10 --warmup 3 > gpurun_out/r02h_bench_c3.json 2>/dev/null; echo "C3 rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r02h_launches_c4.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-raw-key --no-snapshot > /dev/null 2>&1; echo "launches c4 rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r02h_launches_c3.csv \
  python bench.py --config C3 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-snapshot > /dev/null 2>&1; echo "launches c3 rc=$?"
cp profiles/ncu_traffic.json gpurun_out/ncu_traffic.json
for c in C4 C3; do
  n=100000000; [ $c = C3 ] && n=16777216
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum -k regex:k_sweep --clock-control none --csv \
    --log-file gpurun_out/r02h_traffic_$c.csv python scripts/profile_run.py --config $c --max-passes 1000 --pass-csv gpurun_out/r02h_passes_$c.csv > /dev/null 2>&1
  python scripts/ncu_traffic.py --config $c --kernel k_sweep --n $n --launches gpurun_out/r02h_traffic_$c.csv --passes gpurun_out/r02h_passes_$c.csv --out gpurun_out/ncu_traffic.json | grep traffic_over
done
ncu --set full --clock-control none --import-source on -k regex:k_sweep --launch-skip 9 --launch-count 1 -o gpurun_out/r02h_sweep_c4 -f \
  python scripts/profile_run.py --config C4 --max-passes 12 > /dev/null 2>&1; echo "full c4 rc=$?"
