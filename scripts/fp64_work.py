"""fp64 SASS work per leaf cell-stage of a stage kernel from an `ncu --set full` report:
    python scripts/fp64_work.py OUT.json name=REP:CELLS [name=REP:CELLS ...]
count = (op_{dadd,dmul,dfma} .sum.per_cycle_elapsed) x smsp__cycles_elapsed.avg; flops = dadd + dmul + 2 dfma."""
import csv
import io
import json
import subprocess
import sys


def work(rep, cells):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u, v = rows[0], rows[1], rows[2]
    val = lambda k: float(v[h.index(k)].replace(",", ""))   # noqa: E731
    cyc = val("smsp__cycles_elapsed.avg") if "smsp__cycles_elapsed.avg" in h else val("sm__cycles_elapsed.avg")
    d = {op: val(f"smsp__sass_thread_inst_executed_op_{op}_pred_on.sum.per_cycle_elapsed") * cyc / cells
         for op in ("dadd", "dmul", "dfma")}
    ms = val("gpu__time_duration.sum") * {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "second": 1e3, "s": 1e3}[
        u[h.index("gpu__time_duration.sum")]]
    flops = d["dadd"] + d["dmul"] + 2 * d["dfma"]
    return {"fp64_thread_inst_per_cell_stage": d["dadd"] + d["dmul"] + d["dfma"], "flops_per_cell_stage": flops,
            **d, "kernel_ms_under_ncu": ms, "tflops_under_ncu": flops * cells / (ms * 1e-3) / 1e12,
            "fp64_pipe_active_pct": val("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
            "report": rep}


res = {}
for arg in sys.argv[2:]:
    name, spec = arg.split("=")
    rep, cells = spec.split(":")
    try:
        res[name] = work(rep, float(cells))
    except Exception as e:   # noqa: BLE001 -- a missing capture must not lose the others
        res[name] = {"error": repr(e), "report": rep}
res["note"] = ("SASS fp64 op counts per leaf cell-stage from ncu --set full (stage 2 of the 4096^2 sweep); "
               "flops = dadd + dmul + 2 dfma")
json.dump(res, open(sys.argv[1], "w"), indent=1)
print(json.dumps(res, indent=1))
