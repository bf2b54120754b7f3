# Round-2: bench lines of the other configurations (ant = configs[1], sweep points, energies,
# humanoid), short runs without the oracle leg, collected as one JSON per line.
set -u
OUT=gpurun_out/${1:-cfg}
mkdir -p $OUT
: > $OUT/lines.jsonl
run() {  # name, args...
  local n=$1; shift
  timeout 300 python bench.py --steps 100 --warmup 10 --no-cpu-baseline --bulk-updates 0 "$@" > $OUT/$n.json 2> $OUT/$n.err
  python - <<PY >> $OUT/lines.jsonl
import json
d = json.load(open("$OUT/$n.json"))
r = d.get("roofline") or {}
print(json.dumps({"name": "$n", "value": d["value"], "ms": d["ms_per_step"], "e2e": (d.get("e2e") or {}).get("value"),
                  "step_frac": (r.get("step") or {}).get("frac"), "kernel": r.get("kernel"), "frac": r.get("frac")}))
PY
}
run ant --workload ant
run reacher --workload reacher
run humanoid --workload humanoid
run sweep4096 --workload sweep4096
run sweep16384 --workload sweep16384
run sweep16384_cos --workload sweep16384 --energy cos
run sweep16384_dot --workload sweep16384 --energy dot
run sweep4096_cos --workload sweep4096 --energy cos
run netscale_ln --workload netscale --layernorm
run sweep16384_l2sq --workload sweep16384 --energy l2sq
run netscale_l2sq --workload netscale --energy l2sq
cat $OUT/lines.jsonl
