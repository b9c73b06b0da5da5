"""Host regrid phase times averaged over many regrids (GPU box): the shock-bubble (configs[3]) or quadrant
(configs[2]) mesh after the init protocol, then R rounds of 4 CFL-0.5 steps + one regrid with AMR_REGRID_PROF=1;
the library's per-phase lines (stderr) are parsed and averaged over the last R - 2 regrids.

    python scripts/regrid_phases.py sb|q [R]
"""
import os
import re
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import sys
sys.path.insert(0, {root!r})
import paper_2508_05020_b200 as amr, workloads as W
which, R = {which!r}, {R}
cfg = W.shock_bubble(max_patches=100_000) if which == "sb" else W.quadrant(N=512, n=16, levels=3, seed=1)
g = amr.Mesh(cfg)
fn = lambda l, P, Q: W.patch_state(cfg, l, P, Q)
g.set_state(fn)
for _ in range(cfg["levels"] - 1):
    g.regrid(); g.set_state(fn)
for _ in range(R):
    g.steps(4, cfl=0.5)
    g.sync()
    print("== regrid", file=sys.stderr, flush=True)
    g.regrid()
g.close()
"""


def main():
    which = sys.argv[1] if len(sys.argv) > 1 else "sb"
    R = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    env = dict(os.environ, AMR_REGRID_PROF="1")
    r = subprocess.run([sys.executable, "-c", CHILD.format(root=ROOT, which=which, R=R)], capture_output=True,
                       text=True, env=env)
    blocks, cur = [], None
    for ln in r.stderr.splitlines():
        if ln.startswith("== regrid"):
            cur = {}
            blocks.append(cur)
            continue
        m = re.match(r"\s*\[regrid\] (.+?)\s+([0-9.]+) ms", ln)
        if m and cur is not None:
            cur[m.group(1)] = cur.get(m.group(1), 0.0) + float(m.group(2))
    use = blocks[2:]
    avg = defaultdict(float)
    for b in use:
        for k, v in b.items():
            avg[k] += v / len(use)
    print(which, f"{len(use)} regrids, threads={os.environ.get('AMR_HOST_THREADS', 'default')}:",
          {k: round(v, 3) for k, v in avg.items()}, flush=True)
    if r.returncode:
        print(r.stderr[-2000:])


if __name__ == "__main__":
    main()
