# per-stage breakdown (event-bracketed eager profile) for chain vs per-layer schedules
for w in ${WORKLOADS:-ant sweep4096}; do
  for nc in "" 1; do
    echo "== $w NO_CHAIN=$nc"
    env ${nc:+CRL_NO_CHAIN=1} timeout 300 python bench.py --workload $w --steps 50 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["gpu_launches"]); print(json.dumps(d["roofline"].get("stages_us"), indent=0))'
  done
done
