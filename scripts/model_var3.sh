cd $GRAFT_REPO_ROOT
for v in "2 0" "1 1" "1 0"; do set -- $v
  echo "round=$1 rescale=$2"; MODEL_K=8 MODEL_RESCALE=$2 MODEL_MODE=p2p MODEL_ROUND_PASSES=$1 timeout 1200 python scripts/exp_scaling_model.py C4 248.8 0.224 2.6595e10 out 2>&1 | grep "^K="
done
