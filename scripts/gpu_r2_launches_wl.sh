# Round-2: serialized per-kernel durations (ncu launch list, --clock-control none) of one
# workload's bench step, after the same command exits 0 without ncu.  Args: OUT WORKLOAD [extra]
set -u
OUT=gpurun_out/${1:-lw}
WL=${2:-sweep4096}
mkdir -p $OUT
C="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --workload $WL ${3:-}"
$C > $OUT/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv $C > $OUT/ncu.log 2>&1
echo ncu_rc=$?
python - <<PY
import csv, collections
rows = [r for r in csv.reader(open("$OUT/launches.csv")) if len(r) > 10]
h = rows[0]; iname = h.index("Kernel Name"); ival = h.index("Metric Value")
d = collections.OrderedDict()
for r in rows[1:]:
    k = r[iname].split("(")[0][:60]
    d.setdefault(k, []).append(float(r[ival].replace(",", "")))
for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
    print(f"{sum(v)/1e3:10.1f} us total {len(v):5d} launches {sum(v)/len(v)/1e3:9.2f} us avg  {k}")
PY
