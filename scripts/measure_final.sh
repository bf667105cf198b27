# Round-2 final measurements on the final tree (profiles/r02f_*): new tests, bench lines, ncu launch lists, traffic
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_dist.py tests/test_gpu_bench_contract.py -q -k "pilot or bench" > gpurun_out/r02f_newtests.log 2>&1; echo "newtests rc=$?"; tail -3 gpurun_out/r02f_newtests.log
python bench.py --steps 20 --warmup 5 > gpurun_out/r02f_bench_c4.json 2> gpurun_out/r02f_bench_c4.err; echo "c4 rc=$?"
for c in C3 C2 C5 C1; do python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/r02f_bench_$(echo $c | tr C c).json 2>/dev/null; echo "$c rc=$?"; done
python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/r02f_bench_c4_reference.json 2>/dev/null; echo "ref rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r02f_launches_c4.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-raw-key --no-snapshot > /dev/null 2>&1; echo "launches c4 rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r02f_launches_c3.csv \
  python bench.py --config C3 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-snapshot > /dev/null 2>&1; echo "launches c3 rc=$?"
cp profiles/ncu_traffic.json gpurun_out/ncu_traffic.json
for c in C4 C3; do
  n=100000000; [ $c = C3 ] && n=16777216
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum -k regex:k_sweep --clock-control none --csv \
    --log-file gpurun_out/r02f_traffic_$c.csv python scripts/profile_run.py --config $c --max-passes 1000 --pass-csv gpurun_out/r02f_passes_$c.csv > /dev/null 2>&1
  python scripts/ncu_traffic.py --config $c --kernel k_sweep --n $n --launches gpurun_out/r02f_traffic_$c.csv --passes gpurun_out/r02f_passes_$c.csv --out gpurun_out/ncu_traffic.json | grep traffic_over
done
ncu --set full --clock-control none --import-source on -k regex:k_sweep --launch-skip 10 --launch-count 1 -o gpurun_out/r02f_sweep_c3 -f \
  python scripts/profile_run.py --config C3 --max-passes 14 > /dev/null 2>&1; echo "full c3 rc=$?"
