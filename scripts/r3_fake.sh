cd ${GRAFT_REPO_ROOT:-.}
for v in i2 i2fake; do
DITER_LIB=$PWD/variants/v_$v.so ncu --metrics gpu__time_duration.sum -k regex:k_sweep --clock-control none --csv --log-file gpurun_out/r3_fk_$v.csv \
  python scripts/profile_run.py --config C4 --max-passes 12 --pass-csv gpurun_out/r3_fk_${v}_passes.csv > /dev/null 2>&1; echo rc=$?
done
