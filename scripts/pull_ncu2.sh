cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
EXP_WARM=0 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_red.sum,lts__t_sectors_srcunit_tex_op_red_lookup_miss.sum --clock-control none --csv --log-file gpurun_out/push_launches_c4.csv python scripts/exp_pull.py C4 "-1:0" 1 > gpurun_out/push_ncu.log 2>&1; echo "rc=$?"
tail -2 gpurun_out/push_ncu.log
