# Round-2: the whole GPU test suite, then the default bench line and the launch list.
set -u
OUT=gpurun_out/${1:-full}
mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
tail -3 $OUT/pytest_gpu.log
timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > $OUT/bench_netscale.json 2> $OUT/bench_netscale.err
python - <<PY
import json
d = json.load(open("$OUT/bench_netscale.json"))
print(d["value"], d["ms_per_step"], d["e2e"]["value"], d["roofline"]["step"]["frac"])
PY
[ -n "${2:-}" ] && bash scripts/gpu_r2_launches.sh ${1:-full}/ln | tail -22
