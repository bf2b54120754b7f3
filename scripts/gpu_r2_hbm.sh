# Round-2: HBM evidence for the HBM-bound stages: buffer insert (A0), bulk
# relabel sample (A1, 2^22 rows) and Adam (A6) at netscale: dram bytes and durations per launch
# from ncu (after the same bench command exits 0 without ncu).
set -u
OUT=gpurun_out/${1:-hbm}
mkdir -p $OUT
C="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --profile-steps 0"
$C > $OUT/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum \
    --clock-control none -k regex:"relabel_sample_kernel|adam_kernel|buffer_insert_kernel" --launch-skip 18 -c 8 --csv \
    --log-file $OUT/hbm.csv $C > $OUT/ncu.log 2>&1
echo ncu_rc=$?
python - <<PY
import csv, collections
rows = [r for r in csv.reader(open("$OUT/hbm.csv")) if len(r) > 10]
h = rows[0]
ik, im, iv, iu, iid = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit"), h.index("ID")
d = collections.OrderedDict()
for r in rows[1:]:
    d.setdefault((r[iid], r[ik].split("(")[0]), {})[r[im]] = (float(r[iv].replace(",", "")), r[iu])
for (i, k), m in d.items():
    t = m["gpu__time_duration.sum"]
    tus = t[0] / 1e3 if t[1] in ("ns", "nsecond") else t[0]
    def by(name):
        v, u = m[name]
        return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
    rd, wr = by("dram__bytes_read.sum"), by("dram__bytes_write.sum")
    print(f"{k:40s} {tus:9.2f} us  dram read {rd/1e6:8.2f} MB  write {wr/1e6:8.2f} MB  -> {(rd+wr)/tus/1e3:7.1f} GB/s")
PY
