"""Assemble profiles/<TAG>_amr_launches.json (CPU) from the artefacts scripts/amr_profile.sh leaves in gpurun_out/:
the per-kernel launch lists of configs[2] / configs[3] (ncu --metrics gpu__time_duration.sum of amr_launches.py: 4 steps
+ 1 regrid after the init protocol and warm-up; cold-cache, serialised: shares, not absolutes), the AMR step / regrid
times with and without graphs (quick_perf.py amr amr_graphs) and the host regrid phase timers of the profiled regrid
(AMR_REGRID_PROF=1; the timers synchronise the device per phase).

    python scripts/amr_evidence.py TAG
"""
import csv
import io
import json
import re
import sys
from collections import defaultdict


def launches(path):
    lines = [ln for ln in open(path) if ln.startswith('"')]
    agg = defaultdict(lambda: [0, 0.0])
    for r in csv.DictReader(io.StringIO("".join(lines))):
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0]
        v = float(r["Metric Value"].replace(",", ""))
        agg[name][0] += 1
        agg[name][1] += v / 1e3 if r["Metric Unit"] == "ns" else (v if r["Metric Unit"] == "us" else v * 1e3)
    tot = sum(t for _, t in agg.values()) or 1.0
    return {k: {"launches": n, "total_us": t, "mean_us": t / n, "share": t / tot}
            for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])}


def regrid_phases(path):
    """The last block of '[regrid] phase x ms' lines (the profiled regrid)."""
    blocks, cur = [], []
    for ln in open(path):
        m = re.match(r"\s*\[regrid\] (.+?)\s+([0-9.]+) ms", ln)
        if m:
            if m.group(1) == "flags" and cur:
                blocks.append(cur)
                cur = []
            cur.append((m.group(1), float(m.group(2))))
    if cur:
        blocks.append(cur)
    return dict(blocks[-1]) if blocks else {}


def main():
    tag = sys.argv[1]
    g = "gpurun_out"
    out = {"configs2_quadrant": launches(f"{g}/amr_launches_q_{tag}.csv"),
           "configs3_shock_bubble": launches(f"{g}/amr_launches_sb_{tag}.csv"),
           "note": "ncu --metrics gpu__time_duration.sum of scripts/amr_launches.py (4 CFL-0.5 steps + 1 regrid after "
                   "the init protocol and 4 warm-up steps), cold-cache and serialised: shares, not absolutes",
           "step_times": [json.loads(ln) for ln in open(f"{g}/amr_perf_{tag}.log") if ln.startswith("{")],
           "regrid_phases_ms_configs3": regrid_phases(f"{g}/amr_regrid_prof_sb_{tag}.log")}
    json.dump(out, open(f"profiles/{tag}_amr_launches.json", "w"), indent=1)
    print(f"profiles/{tag}_amr_launches.json")


if __name__ == "__main__":
    main()
