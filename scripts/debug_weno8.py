"""Debug: WENO5-char sweep on white noise -- cells where the oracle's state is NaN: is the GPU's state there
non-physical too?  python scripts/debug_weno8.py (GPU box)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2508_05020_b200 as amr, workloads as W
from tests.test_gpu_fullsize import block_oracle
for n, N in ((16, 256), (8, 256)):
    cfg = W.sweep(N=N, n=n, scheme="weno5", seed=7); cfg.update(check_positivity=0, characteristic=1)
    g = amr.Mesh(cfg); g.set_state(U=W.level0_state(cfg).reshape(-1, 4, n, n))
    _, lam = g.diagnostics(); dt = 0.3 / lam; g.step(dt=dt)
    U = g.get_state(as_dict=False, indices=np.array([0], np.int32))[0]; g.close()
    Uo = block_oracle(cfg, 0, 0, dt)
    bad = np.isnan(Uo).any(axis=0)
    r, m, w, E = U
    p = 0.4 * (E - 0.5 * (m * m + w * w) / r)
    phys = (r > 0) & (p > 0) & np.isfinite(U).all(axis=0)
    print(N, n, 'oracle NaN cells', bad.sum(), 'GPU physical there', (phys & bad).sum(), 'GPU rho/p there', r[bad][:4], p[bad][:4])
    print('   oracle finite cells where the GPU is non-physical', (~phys & ~bad).sum())
