"""Summarise a round-2 `ncu --set full` capture (scripts/gpu_r2_ncufull.sh) of the netscale step:
per kernel launch the duration, DRAM bytes and pipe utilisations; updates
profiles/ncu_traffic.json["netscale/bf16"] (bench stage -> DRAM bytes per launch, the
`roofline.traffic` bench.py reports).

    python scripts/summarize_ncu_r2.py gpurun_out/nf/full.ncu-rep profiles/round2/ncu_full_netscale.txt
"""
import csv
import io
import json
import os
import subprocess
import sys

STAGE = {"tc_grad2p_kernel": "grad_pair", "tc_stats_kernel": "lse_fused", "tc_dwg_kernel": "dw_db_grouped",
         "tc_pdw_kernel": "dw_db_pairs", "adam_kernel": "adam", "grad_merge2_kernel": "grad_merge"}
METRICS = [("gpu__time_duration.sum", "us", 1e-3),
           ("dram__bytes_read.sum", "MB rd", 1e-6), ("dram__bytes_write.sum", "MB wr", 1e-6),
           ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "% tensor", 1),
           ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "% XU", 1),
           ("sm__issue_active.avg.pct_of_peak_sustained_elapsed", "% issue", 1),
           ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "% smem lsu", 1),
           ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "% L2", 1),
           ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "% DRAM", 1)]
UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1.0, "usecond": 1e3, "msecond": 1e6,
        "ns": 1.0, "us": 1e3, "ms": 1e6}


def main(rep, out):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    lines = ["ncu --set full --clock-control none (netscale step, configs[4], W = 1, bf16); cold caches between",
             "replays, so absolute times exceed the in-graph ones: compare shares and pipe utilisations.", ""]
    traffic = {}
    for r in data:
        name = r[hdr.index("Kernel Name")]
        short = name.split("(")[0].replace("void ", "").split("::")[-1].split("<")[0]
        vals = []
        for m, label, sc in METRICS:
            if m not in hdr:
                continue
            i = hdr.index(m)
            v = float(r[i].replace(",", "")) * UNIT.get(units[i], 1.0) if r[i] else float("nan")
            if m.startswith("gpu__time"):
                v = v * 1e-3   # ns -> us
            elif m.startswith("dram__bytes"):
                v = v * 1e-6   # bytes -> MB
            vals.append(f"{label} {v:9.2f}")
        lines.append(f"{name.split('(')[0][:60]:60s} " + "  ".join(vals))
        if short in STAGE:
            rd = float(r[hdr.index("dram__bytes_read.sum")].replace(",", "")) * UNIT.get(units[hdr.index("dram__bytes_read.sum")], 1)
            wr = float(r[hdr.index("dram__bytes_write.sum")].replace(",", "")) * UNIT.get(units[hdr.index("dram__bytes_write.sum")], 1)
            traffic.setdefault(STAGE[short], int(rd + wr))
    open(out, "w").write("\n".join(lines) + "\n")
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "profiles", "ncu_traffic.json")
    db = json.load(open(path)) if os.path.exists(path) else {}
    db.setdefault("netscale/bf16", {}).update(traffic)
    json.dump(db, open(path, "w"), indent=1, sort_keys=True)
    print("\n".join(lines))
    print(traffic)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
