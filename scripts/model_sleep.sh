cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -k "p2p or ipc" > gpurun_out/p2p3.log 2>&1; echo rc=$?; tail -2 gpurun_out/p2p3.log
for sl in 0 -1; do echo "sleep=$sl"; MODEL_SLEEP=$sl MODEL_MODE=p2p MODEL_ROUND_PASSES=2 timeout 1200 python scripts/exp_scaling_model.py C4 248.8 0.224 2.6595e10 out > gpurun_out/msleep_$sl.txt 2>&1; grep "^K=" gpurun_out/msleep_$sl.txt; done
