# Round-2 GPU pass: the whole -m gpu suite (full-scale oracle comparison included), then
# the per-launch DRAM traffic of k_scatter over one solve of C4 and C3 (ncu metrics).
cd $GRAFT_REPO_ROOT
timeout 3600 python -m pytest tests -m gpu -v -x --timeout 2400 -s > gpurun_out/gpu_all.log 2>&1; echo tests_rc=$?
grep -E "passed|failed|H - X_ref" gpurun_out/gpu_all.log | tail -5
for C in C4 C3; do
  timeout 600 python scripts/profile_run.py --config $C --max-passes 1000 --pass-csv gpurun_out/passes_$C.csv > gpurun_out/plain_$C.log 2>&1 && \
  timeout 1800 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum -k regex:k_scatter --clock-control none --csv --log-file gpurun_out/traffic_$C.csv python scripts/profile_run.py --config $C --max-passes 1000 > gpurun_out/ncu_traffic_$C.log 2>&1
  echo ncu_$C=$?
done
