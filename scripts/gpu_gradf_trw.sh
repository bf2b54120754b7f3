for d in ${DBGS:-40 44}; do echo "== dbg=$d"; CRL_GF_DBG=$d timeout 300 python bench.py --workload ${W:-sweep16384} --steps 1 --warmup 1 --profile-steps 0 --no-cpu-baseline --no-e2e 2>&1 | grep GF_TRW | tail -512 | grep -v "^GF_TRW 64" | python -c '
import sys,collections
d=collections.defaultdict(dict)
for l in sys.stdin:
  _,bx,t,w,v=l.split(); d[(int(bx),int(t))][int(w)]=int(v)
for k in sorted(d):
  v=[d[k][w] for w in range(16)]; m=min(v)
  print(k, "min", m, "spread", max(v)-m, "per-warp", [x-m for x in v])
'
done
