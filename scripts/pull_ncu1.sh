cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
EXP_WARM=0 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/pull_launches_c4.csv python scripts/exp_pull.py C4 "1:0" 1 > gpurun_out/pull_ncu.log 2>&1; echo "rc=$?"
tail -3 gpurun_out/pull_ncu.log
