# clock64 trace of tc_gradf CTAs (0,0) and (R/2,0): 1 S issued, 2 back issued, 3 epi S ready, 4 W done, 5 readout done, 6 dB ready
for d in ${DBGS:-8 24}; do
CRL_GF_DBG=$d timeout 300 python bench.py --workload ${W:-sweep16384} --steps 1 --warmup 3 --profile-steps 0 --no-cpu-baseline --no-e2e 2>&1 | grep GF_TRACE | tail -192 | python -c '
import sys,collections
d=collections.defaultdict(dict)
for l in sys.stdin:
  _,bx,k,t,v=l.split(); d[(int(bx),int(t))][int(k)]=int(v)
print("dbg='$d' (cta, t): S_iss back_iss epiS Wdone rdone dBready")
for t in sorted(d): print(t, [d[t].get(k) for k in range(1,7)])
'
done
