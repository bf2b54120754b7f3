# Round-2 knob sweep: the default (netscale) bench line under each value of an environment knob.
#   bash scripts/gpu_r2_sweep.sh OUT KNOB "v1 v2 ..."
set -u
OUT=gpurun_out/${1:-sw}
KNOB=${2:-CRL_DW_SPLITS}
mkdir -p $OUT
for v in ${3:-1 2 4 8}; do
  env $KNOB=$v timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > $OUT/b_$v.json 2> $OUT/b_$v.err
  python - <<PY
import json
d = json.load(open("$OUT/b_$v.json"))
s = d["roofline"]["stages_us"]
print("$KNOB=$v", d["value"], d["ms_per_step"], {k: s[k] for k in ("dw_db_grouped", "adam", "grad_pair", "lse_fused") if k in s})
PY
done
