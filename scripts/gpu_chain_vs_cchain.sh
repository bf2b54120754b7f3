# fwd/bwd chain variant comparison across batch sizes (per-stage us + step ms)
b() { timeout 300 python bench.py --workload $1 --steps ${STEPS:-300} --warmup 20 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["config"]["workload"], d["ms_per_step"], d["value"], json.dumps(d["roofline"].get("stages_us")))'; }
for w in sweep2048 sweep4096; do echo "== $w default"; b $w; echo "== $w CRL_CHAIN"; CRL_CHAIN=1 b $w; done
echo "== sweep8192 CRL_CCHAIN"; CRL_CCHAIN=1 b sweep8192
