"""Summarise an ncu measurement pass (scripts/gpu_round1_measure.sh output) into profiles/.

    python scripts/summarize_ncu.py gpurun_out/r1 profiles/round1

Writes, per captured workload: <dst>/launches_<w>.txt (per-launch device times from the
--metrics gpu__time_duration.sum pass: cold-cache, serialised -- compare SHARES), and
<dst>/ncu_full_<w>.txt (per kernel: duration, DRAM bytes, pipe utilisation from --set full);
and updates profiles/ncu_traffic.json, the per-launch DRAM traffic bench.py reports as
roofline.traffic (key "<workload>/<precision>" -> {bench stage: bytes per launch}).
Needs the ncu CLI (reads the .ncu-rep files with `ncu -i`)."""
import csv
import io
import json
import os
import subprocess
import sys

# bench.py stage name -> the kernel that stage launches (the dominant one of the stage)
STAGE_KERNEL = {
    "mlp_fwd_cchain": "tc_cchain_kernel<0>", "mlp_bwd_cchain": "tc_cchain_kernel<1>",
    "mlp_fwd_chain": "tc_chain_kernel<0>", "mlp_bwd_chain": "tc_chain_kernel<1>",
    "lse_fused": "tc_stats_kernel", "grad_fused": "tc_gradf_kernel", "dw_db_grouped": "tc_dwg_kernel",
}
UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def launches(src, w, dst):
    path = os.path.join(src, f"launches_{w}.csv")
    if not os.path.exists(path):
        return
    rows = [r for r in csv.reader(open(path)) if len(r) > 10][1:]
    tot = sum(float(r[14]) for r in rows) / 1000
    with open(os.path.join(dst, f"launches_{w}.txt"), "w") as f:
        f.write(f"# ncu --metrics gpu__time_duration.sum --clock-control none ({w}, bf16): {len(rows)} launches, "
                f"{tot:.2f} us summed (serialised, no programmatic-launch overlap: compare shares)\n")
        for r in rows:
            t = float(r[14]) / 1000
            f.write(f"{t:9.2f} us  {100 * t / tot:5.1f}%  grid={r[8]:>14}  {r[4][:110]}\n")


def full(src, w, dst, traffic):
    rep = os.path.join(src, f"{w}_full.ncu-rep")
    if not os.path.exists(rep):
        return
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, u = rows[0], rows[1]
    want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
            "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__grid_size", "launch__registers_per_thread"]
    idx = {k: h.index(k) for k in want if k in h}
    ki = h.index("Kernel Name")
    with open(os.path.join(dst, f"ncu_full_{w}.txt"), "w") as f:
        f.write(f"# ncu --set full --clock-control none ({w}, bf16): one line per captured launch\n")
        for r in rows[2:]:
            f.write(r[ki][:70] + "\n")
            for k, i in idx.items():
                f.write(f"    {k:62s} {r[i]} {u[i]}\n")
            rd = float(r[idx["dram__bytes_read.sum"]]) * UNIT.get(u[idx["dram__bytes_read.sum"]], 1.0)
            wr = float(r[idx["dram__bytes_write.sum"]]) * UNIT.get(u[idx["dram__bytes_write.sum"]], 1.0)
            for stage, kern in STAGE_KERNEL.items():
                if kern in r[ki].replace(" ", ""):
                    traffic.setdefault(f"{w}/bf16", {})[stage] = round(rd + wr)


def main():
    src, dst = sys.argv[1], sys.argv[2]
    os.makedirs(dst, exist_ok=True)
    tpath = os.path.join(os.path.dirname(dst.rstrip("/")), "ncu_traffic.json")
    traffic = json.load(open(tpath)) if os.path.exists(tpath) else {}
    for w in ("ant", "sweep16384", "sweep4096"):
        launches(src, w, dst)
        full(src, w, dst, traffic)
    with open(tpath, "w") as f:
        json.dump(traffic, f, indent=1, sort_keys=True)
    print(json.dumps(traffic, indent=1))


if __name__ == "__main__":
    main()
