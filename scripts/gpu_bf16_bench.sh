# bf16 parity suite, then steps/s on the sweep workloads (default schedule)
python -m pytest tests -m gpu -x -q -k "bf16" 2>&1 | tail -4
for w in ${WORKLOADS:-ant sweep4096 sweep16384}; do
  timeout 300 python bench.py --workload $w --steps ${STEPS:-300} --warmup 20 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["config"]["workload"], d["ms_per_step"], d["value"], d["gpu_launches"], json.dumps(d["roofline"].get("stages_us")))'
done
