# Round-2 quick loop: a pytest subset (-k expression), the default bench line, optional ncu.
set -u
OUT=gpurun_out/${1:-q}
K=${2:-grad2}
NCU=${3:-}
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q -x -k "$K" > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
tail -3 $OUT/pytest_gpu.log
timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > $OUT/bench_netscale.json 2> $OUT/bench_netscale.err
python - <<PY
import json
d = json.load(open("$OUT/bench_netscale.json"))
print(d["value"], d["ms_per_step"], d["e2e"]["value"], d["roofline"]["step"]["frac"])
print({k: v for k, v in d["roofline"]["stages_us"].items()})
PY
if [ -n "$NCU" ]; then bash scripts/gpu_r2_ncu.sh $1/ncu "$NCU" 2 > /dev/null 2>&1; ls $OUT/ncu; fi
