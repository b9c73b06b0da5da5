"""A/B of amr_config.stage_kernel on the AMR configs (kernel timing through the library's CUDA events):
    python scripts/amr_ab_variant.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_05020_b200 as amr  # noqa: E402
import workloads as W  # noqa: E402

for name, cfg0 in [("quadrant", W.quadrant(N=512, n=16, levels=3, seed=1)), ("shock_bubble", W.shock_bubble())]:
    for v in (1, 0, 1, 0):
        cfg = dict(cfg0, stage_kernel=v)
        g = amr.Mesh(cfg)
        fn = lambda l, P, Q: W.patch_state(cfg, l, P, Q)   # noqa: E731
        g.set_state(fn)
        for _ in range(cfg["levels"] - 1):
            g.regrid()
            g.set_state(fn)
        for s in range(4):
            g.step(cfl=0.5)
        g.set_kernel_timing(True)
        g.reset_stats()
        for s in range(6):
            g.step(cfl=0.5)
        g.sync()
        st = g.stats()
        print(name, "stage_kernel", v, "stage ms %.4f" % (st["stage_ms"] / max(1, st["stage_timed"])),
              "leaves", st["leaves"], "G cell/s %.2f" % (st["stage_cells"] / (st["stage_ms"] * 1e-3) / 1e9), flush=True)
        g.close()
