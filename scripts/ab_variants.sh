cd $GRAFT_REPO_ROOT
for c in C4 C3; do for v in base tp base tp; do
  echo "$c $v $(DITER_LIB=$PWD/variants/v_$v.so timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_per_step'],2), d['roofline']['kernel_shares']['k_scatter'], round(d['roofline']['atomic_issue']['frac'],3))")"
done; done
