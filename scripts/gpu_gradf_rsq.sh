# tc_gradf: share of logit pairs whose rsqrt runs on the FMA pipe (rebuilds tc_gradf.cu per variant)
cd paper_2408_11052_b200/csrc
for k in ${KS:-0 1 2 3 4}; do
  touch tc_gradf.cu; make NVFLAGS_EXTRA="-DCRL_GF_RSQ_EMU=$k" > /dev/null 2>&1 || { echo "build $k failed"; continue; }
  (cd ../..; for w in ${WS:-sweep16384 sweep4096}; do echo -n "rsq_emu=$k $w "; timeout 200 python bench.py --workload $w --steps 100 --warmup 10 --no-cpu-baseline --no-e2e --bulk-updates 0 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); s=d["roofline"].get("stages_us"); print(d["ms_per_step"], s.get("grad_fused"))'; done)
done
(cd ../..; timeout 200 python -m pytest tests -m gpu -x -q -k "bf16_small or fused_chain or stats_paths" 2>&1 | tail -1)
