# tc_gradf timing ablations (parity is NOT expected under CRL_GF_DBG)
for d in ${DBGS:-0 1 2 3 4 7}; do
  echo -n "dbg=$d "; CRL_GF_DBG=$d timeout 300 python bench.py --workload ${W:-sweep16384} --steps 100 --warmup 10 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); s=d["roofline"].get("stages_us"); print(d["ms_per_step"], s.get("grad_fused"), s.get("lse_fused"))'
done
