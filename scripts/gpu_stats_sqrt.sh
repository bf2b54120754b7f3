# tc_stats: share of logit pairs whose sqrt runs on the FMA pipe (rebuilds tc_stats.cu per variant)
cd paper_2408_11052_b200/csrc
for k in ${KS:-0 1 2 3 4}; do
  touch tc_stats.cu; make NVFLAGS_EXTRA="-DCRL_ST_SQRT_EMU=$k" > /dev/null 2>&1 || { echo "build $k failed"; continue; }
  (cd ../..; echo -n "sqrt_emu=$k "; timeout 200 python bench.py --workload ${W:-sweep16384} --steps 100 --warmup 10 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); s=d["roofline"].get("stages_us"); print(d["ms_per_step"], s.get("lse_fused"), s.get("grad_fused"))')
done
(cd ../..; timeout 120 python -m pytest tests -m gpu -x -q -k "bf16_sweep4096 or bf16_small or stats_paths" 2>&1 | tail -1)
