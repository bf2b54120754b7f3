for sp in ${SPLITS:-1 2 4 8 16}; do
  echo -n "splits=$sp "; CRL_GF_SPLITS=$sp timeout 300 python bench.py --workload ${W:-sweep16384} --steps 100 --warmup 10 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); s=d["roofline"].get("stages_us"); print(d["ms_per_step"], s.get("grad_fused"), s.get("lse_fused"))'
done
