#!/usr/bin/env python
"""NEXT #1: fusion-granularity study on B200 -- the GPU analogue of the paper's task-fusion result
(18x) and GPU-kernel result (9.7x).

For patch sizes n = 8/16/32/64 on a periodic noise field (BASELINE configs[4] distributions), Central4 (and
WENO5-char at n = 16/32), each stage organisation of amr_config.stage_kernel is timed with and without CUDA
graphs (use_graphs):
  0 fused (default: persistent TMA kernel for n >= 32), 1 fused one-CTA-per-tile, 2 unfused (4 kernels, HBM
  intermediates), 3 one fused launch per leaf patch (the task-per-patch analogue).
Time: CUDA events on the library stream around K steps after W warm-up steps (graph capture in the warm-up);
each timed step starts from the pristine state (untimed restore).  Writes profiles/<tag>_fusion_study.json.

    python scripts/fusion_study.py [--N 2048] [--steps 3] [--tag r1]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2508_05020_b200 as amr  # noqa: E402
import workloads as W  # noqa: E402


def time_config(N, n, scheme, variant, graphs, steps, warmup, stream):
    cfg = W.sweep(N=N, n=n, scheme=scheme, seed=7)
    cfg.update(check_positivity=0, stage_kernel=variant, use_graphs=graphs, characteristic=1)
    g = amr.Mesh(cfg, stream=stream)
    U0 = torch.from_numpy(W.level0_state(cfg).reshape(-1, 4, n, n)).cuda()
    idx = np.arange(U0.shape[0], dtype=np.int32)
    g.set_state_device(U0, indices=idx)
    _, lam = g.diagnostics()
    dt = 0.3 / lam
    for _ in range(warmup):
        g.set_state_device(U0, indices=idx)
        g.steps(1, dt=dt)
    torch.cuda.synchronize()
    g.reset_stats()
    ms = 0.0
    for _ in range(steps):
        g.set_state_device(U0, indices=idx)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        g.steps(1, dt=dt)
        e1.record(stream)
        e1.synchronize()
        ms += e0.elapsed_time(e1)
    st = g.stats()
    g.close()
    cells = N * N
    return {"ms_per_step": ms / steps, "cell_updates_per_s": cells * 3 * steps / (ms / 1e3),
            "launches_per_step": st["launches"] / steps}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--N", type=int, default=2048)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--tag", default="r1")
    ap.add_argument("--per-patch-max", type=int, default=4096,
                    help="skip the one-launch-per-patch organisation above this many patches (launch-bound: ~5 us each)")
    a = ap.parse_args()
    from paper_2508_05020_b200 import build as B
    B.build()
    stream = torch.cuda.Stream()
    rows = []
    plan = [("central4", n) for n in (8, 16, 32, 64)] + [("weno5", n) for n in (16, 32)]
    for scheme, n in plan:
        for variant in (0, 1, 2, 3):
            for graphs in (0, 1):
                if variant == 3 and (a.N // n) ** 2 > a.per_patch_max:
                    rows.append(dict(scheme=scheme, n=n, stage_kernel=variant, use_graphs=graphs, ms_per_step=None,
                                     skipped=f"{(a.N // n) ** 2} patches > --per-patch-max"))
                    continue
                r = time_config(a.N, n, scheme, variant, graphs, a.steps, a.warmup, stream)
                r.update(scheme=scheme, n=n, stage_kernel=variant, use_graphs=graphs)
                rows.append(r)
                print(f"{scheme:9s} n={n:2d} variant={variant} graphs={graphs}: {r['ms_per_step']:9.3f} ms/step "
                      f"{r['cell_updates_per_s'] / 1e9:7.2f} G cell-updates/s  {r['launches_per_step']:.0f} launches/step",
                      flush=True)
    out = {"workload": f"BASELINE configs[4] noise field, {a.N}^2 periodic, 1 level, fixed dt (CFL 0.3)",
           "timing": "CUDA events on the library stream, per SSP-RK3 step, mean of %d steps after %d warm-up" % (a.steps, a.warmup),
           "paper_context": {"task_fusion_speedup": "18x (P:L277, Regent/Legion, CPU tasks)",
                             "ssprk3Stage_gpu_speedup": "9.7x = 347.0 ms CPU -> 35.7 ms GPU at 2560^2 (P:L285)"},
           "rows": rows}
    for scheme, n in plan:
        sel = {(r["stage_kernel"], r["use_graphs"]): r["ms_per_step"] for r in rows if r["scheme"] == scheme and r["n"] == n}
        best = min(sel[(0, 0)], sel[(0, 1)])
        pp = sel[(3, 0)] is not None
        out.setdefault("speedups", []).append({
            "scheme": scheme, "n": n,
            "fused_vs_unfused": sel[(2, 0)] / sel[(0, 0)],
            "fused_vs_unfused_graphs": sel[(2, 1)] / sel[(0, 1)],
            "fused_vs_per_patch_launches": sel[(3, 0)] / sel[(0, 0)] if pp else None,
            "fused_vs_per_patch_graph": sel[(3, 1)] / best if pp else None,
            "graphs_on_per_patch": sel[(3, 0)] / sel[(3, 1)] if pp else None})
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", f"{a.tag}_fusion_study.json"), "w") as f:
        json.dump(out, f, indent=1)
    for s in out["speedups"]:
        print(s)


if __name__ == "__main__":
    main()
