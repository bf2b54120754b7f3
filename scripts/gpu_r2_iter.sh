# Round-2 iteration pass: GPU tests (stop at first failure) and the default bench line.
set -u
OUT=gpurun_out/${1:-it}
mkdir -p $OUT
timeout 1200 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > $OUT/bench_netscale.json 2> $OUT/bench_netscale.err
tail -4 $OUT/pytest_gpu.log
python - <<PY
import json
d = json.load(open("$OUT/bench_netscale.json"))
print(d["value"], d["ms_per_step"], d["e2e"]["value"], d["roofline"]["step"]["frac"])
print({k: v for k, v in d["roofline"]["stages_us"].items()})
PY
