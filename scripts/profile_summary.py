"""Write the judged profile summaries under profiles/ from gpurun_out/ artefacts.

    python scripts/profile_summary.py TAG [rep ...]

 - profiles/<TAG>_ncu_summary.jsonl : key raw metrics of each `ncu --set full` report given
 - profiles/<TAG>_launches.json     : per-kernel launch counts, total / mean duration and share of the launch list
   (gpurun_out/launches_<TAG>.csv, the `--metrics gpu__time_duration.sum` pass; cold-cache, serialised)
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

KEYS = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "lts__t_sector_hit_rate.pct", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "sm__cycles_elapsed.avg", "dram__throughput.avg.pct_of_peak_sustained_elapsed"]


def raw_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u, v = rows[0], rows[1], rows[2]
    d = {k: (v[h.index(k)] + (" " + u[h.index(k)] if u[h.index(k)] else "")) for k in KEYS if k in h}
    d["stalls_per_issue"] = {k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""):
                             float(v[i]) for i, k in enumerate(h)
                             if k.startswith("smsp__average_warps_issue_stalled") and k.endswith("per_issue_active.ratio")
                             and v[i] and float(v[i]) > 0.05}
    return d


def launches(path):
    agg = defaultdict(lambda: [0, 0.0])
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(io.StringIO("".join(lines))):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0]
        ns = float(r["Metric Value"].replace(",", "")) * (1000.0 if r["Metric Unit"] == "us" else 1.0)
        agg[name][0] += 1
        agg[name][1] += ns
    tot = sum(v[1] for v in agg.values())
    return {k: {"launches": v[0], "total_us": v[1] / 1e3, "mean_us": v[1] / v[0] / 1e3, "share": v[1] / tot}
            for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])}


if __name__ == "__main__":
    tag = sys.argv[1]
    os.makedirs("profiles", exist_ok=True)
    reps = sys.argv[2:]
    if reps:
        with open(f"profiles/{tag}_ncu_summary.jsonl", "w") as f:
            for rep in reps:
                try:
                    m = raw_metrics(rep)
                except Exception as e:   # noqa: BLE001 -- a missing capture must not lose the others
                    m = {"error": repr(e)}
                f.write(json.dumps({os.path.basename(rep).replace(".ncu-rep", ""): m}) + "\n")
    lp = f"gpurun_out/launches_{tag}.csv"
    if os.path.exists(lp):
        json.dump(launches(lp), open(f"profiles/{tag}_launches.json", "w"), indent=1)
    print("written", tag)
