# A/B of the stored-W gradient path (side 1 as W^T Phi) against both sides in the pair pass.
set -u
OUT=gpurun_out/${1:-wsym}
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q -x -k "${2:-stored_w or grad2 or repr256 or l2sq or full_size}" > $OUT/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> $OUT/pytest_gpu.log
tail -3 $OUT/pytest_gpu.log
for v in on off on off; do
  VAR=${ABVAR:-CRL_NO_G2_WSYM}   # the knob that turns the variant under test off
  if [ $v = off ]; then export $VAR=1; else unset $VAR; fi
  timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > $OUT/bench_$v.json 2> $OUT/bench_$v.err
  python - <<PY
import json
d = json.load(open("$OUT/bench_$v.json"))
print("$v", d["value"], d["ms_per_step"], d["e2e"]["value"], d["clocks"]["sm_mhz"])
print({k: v for k, v in d["roofline"]["stages_us"].items() if v > 20})
PY
done
unset ${ABVAR:-CRL_NO_G2_WSYM}
bash scripts/gpu_r2_launches_wl.sh ${1:-wsym}/lw_on netscale | head -14
env ${ABVAR:-CRL_NO_G2_WSYM}=1 bash scripts/gpu_r2_launches_wl.sh ${1:-wsym}/lw_off netscale | head -8
