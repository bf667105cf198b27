cd $GRAFT_REPO_ROOT
for v in base tail base tail; do
  echo "$v $(DITER_LIB=$PWD/variants/v_$v.so timeout 300 python bench.py --config C4 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-raw-key 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print(round(d['ms_per_step'],3), round(r['kernel_shares']['k_scatter'],3), round(r['avg_launch_ms']*d['passes_per_solve'],2), d['normalized_iterations'])")"
done
