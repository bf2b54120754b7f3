# small-batch knob sweep (Ant / Reacher): fused-gradient split count
cd $GRAFT_REPO_ROOT
for w in ant reacher; do
  for kv in "X=0" "CRL_GF_SPLITS=1" "CRL_GF_SPLITS=2"; do
    echo "$w $kv $(env $kv timeout 300 python bench.py --workload $w --steps 300 --warmup 10 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["roofline"]["stages_us"].get("grad_fused"))')"
  done
done
