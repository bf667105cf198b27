# Round-2 profiles of the sweep launch configuration (C4, C3): launch list of the bench
# command, per-launch DRAM traffic of k_sweep over one solve, --set full of dense sweeps.
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-raw-key --no-snapshot > gpurun_out/pb_c4.json 2>/dev/null; echo "bench rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r02s_launches_c4.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-raw-key --no-snapshot > gpurun_out/ncu_launch_c4.log 2>&1; echo "launches rc=$?"
for c in C4 C3; do
  n=100000000; [ $c = C3 ] && n=16777216
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum -k regex:k_sweep --clock-control none --csv \
    --log-file gpurun_out/r02s_traffic_$c.csv python scripts/profile_run.py --config $c --max-passes 1000 --pass-csv gpurun_out/r02s_passes_$c.csv > gpurun_out/ncu_tr_$c.log 2>&1; echo "traffic $c rc=$?"
  python scripts/ncu_traffic.py --config $c --kernel k_sweep --n $n --launches gpurun_out/r02s_traffic_$c.csv --passes gpurun_out/r02s_passes_$c.csv --out gpurun_out/ncu_traffic.json | head -8
done
ncu --set full --clock-control none --import-source on -k regex:k_sweep --launch-skip 4 --launch-count 2 -o gpurun_out/r02s_sweep_c4 -f \
  python scripts/profile_run.py --config C4 --max-passes 8 > gpurun_out/ncu_full_c4.log 2>&1; echo "full c4 rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_sweep --launch-skip 10 --launch-count 1 -o gpurun_out/r02s_sweep_c3 -f \
  python scripts/profile_run.py --config C3 --max-passes 14 > gpurun_out/ncu_full_c3.log 2>&1; echo "full c3 rc=$?"
