# tc_pdw ablations at netscale (CRL_PDW_DBG bits: 1 no bias reads, 2 no MMA, 4 no TMA loads);
# serialized per-launch times from the ncu launch list (the dW launch is the second tc_pdw per step)
set -u
OUT=gpurun_out/${1:-pdwabl}
mkdir -p $OUT
for d in ${DBGS:-0 1 2 4 5 6 7}; do
  C="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --bulk-updates 0 --profile-steps 0"
  CRL_PDW_DBG=$d ncu --metrics gpu__time_duration.sum --clock-control none -k regex:tc_pdw --csv \
      --log-file $OUT/l$d.csv $C > /dev/null 2>&1
  python - <<PY
import csv
rows = [r for r in csv.reader(open("$OUT/l$d.csv")) if len(r) > 10]
h = rows[0]; iv = h.index("Metric Value")
t = [float(r[iv].replace(",", "")) / 1e3 for r in rows[1:]]
print("dbg $d", "gemm", round(sum(t[0::2]) / len(t[0::2]), 1), "dW", round(sum(t[1::2]) / len(t[1::2]), 1))
PY
done
