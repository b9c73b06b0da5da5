"""Quick performance probe (GPU box): stage-kernel times of the configs[4] sweep rows and the AMR step times of
configs[2] / configs[3], through bench.py's own measurement functions, one compact JSON line per item.

    python scripts/quick_perf.py [sweep] [amr] [n=16,8] [schemes=weno5_char,central4] [N=4096]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import bench  # noqa: E402
import workloads as W  # noqa: E402


def stage_time(X, n, scheme, char, N=4096, steps=3):
    torch = X.torch
    cfg = W.sweep(N=N, n=n, scheme=scheme, seed=7)
    cfg.update(check_positivity=0, characteristic=char)
    mesh = X.mesh(cfg)
    U0 = torch.from_numpy(W.level0_state(cfg)).cuda().reshape(-1, 4, n, n).contiguous()
    torch.cuda.synchronize()
    idx = np.arange(U0.shape[0], dtype=np.int32)
    mesh.set_state_device(U0, indices=idx)
    _, lam = mesh.diagnostics()
    dt = 0.3 / lam
    mesh.steps(1, dt=dt)
    mesh.reset_stats()
    mesh.set_kernel_timing(True)
    for _ in range(steps):
        mesh.set_state_device(U0, indices=idx)
        mesh.steps(1, dt=dt)
    torch.cuda.synchronize()
    st = mesh.stats()
    mesh.close()
    ms = st["stage_ms"] / max(1, st["stage_timed"])
    rate = st["stage_cells"] / max(1, st["stage_timed"]) / (ms / 1e3)
    out = {"n": n, "N": N, "scheme": scheme + ("_char" if scheme == "weno5" and char else ""), "stage_ms": round(ms, 4),
           "G_cell_stage_per_s": round(rate / 1e9, 3)}
    if scheme == "central4":
        out["hbm_frac"] = round(rate * bench.BYTES_PER_CELL_STAGE / 1e9 / bench.peaks()[0], 4)
    elif char:
        out["fp64_issue_frac"] = round(bench.fp64_work("weno5_char", n)["fp64_thread_inst_per_cell_stage"] * rate /
                                       (148 * 64 * 1.965e9), 4)
    return out


def main():
    args = sys.argv[1:]
    opts = dict(a.split("=", 1) for a in args if "=" in a)
    what = [a for a in args if "=" not in a] or ["sweep", "amr"]
    X = bench.Ctx()
    if "sweep" in what:
        for n in [int(x) for x in opts.get("n", "16,8").split(",")]:
            for sc in opts.get("schemes", "weno5_char").split(","):
                scheme, char = ("weno5", 1) if sc == "weno5_char" else (("weno5", 0) if sc == "weno5_comp" else (sc, 1))
                print(json.dumps(stage_time(X, n, scheme, char, N=int(opts.get("N", 4096)))), flush=True)
    if "amr" in what:
        q = bench.measure_quadrant(X, None)
        print(json.dumps({"quadrant": {k: q[k] for k in ("ms_per_step", "regrid_ms_per_call", "step_ms_without_regrid",
                                                           "windows_ms_per_step")}}), flush=True)
        sb = bench.measure_amr(X, W.shock_bubble(max_patches=100_000), "configs[3]")
        print(json.dumps({"shock_bubble": {k: sb[k] for k in ("ms_per_step", "regrid_ms_per_call",
                                                               "step_ms_without_regrid", "windows_ms_per_step")}}),
              flush=True)
    if "amr_graphs" in what:
        q = bench.measure_quadrant(X, None, use_graphs=1)
        print(json.dumps({"quadrant_graphs": {k: q[k] for k in ("ms_per_step", "regrid_ms_per_call",
                                                                  "step_ms_without_regrid")}}), flush=True)


if __name__ == "__main__":
    main()
