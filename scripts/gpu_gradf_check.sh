# fused-gradient parity + per-stage timings at the sweep sizes
timeout 600 python -m pytest tests -m gpu -x -q -k "bf16 or fused or stats" 2>&1 | tail -3
for w in ${WORKLOADS:-sweep16384 sweep4096 ant}; do
  timeout 300 python bench.py --workload $w --steps ${STEPS:-300} --warmup 20 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["config"]["workload"], d["ms_per_step"], d["value"], json.dumps(d["roofline"].get("stages_us")))'
done
