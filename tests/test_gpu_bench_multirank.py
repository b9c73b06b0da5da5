"""The N > 1 bench path (torchrun, one process per rank, max-over-ranks timing, slab partition, e2e through the
public API) run on one GPU over the host-collective test transport (AMR_BENCH_HOST_COMM=1): the JSON line must be
complete and the per-step conservation drift of the 2-rank periodic sweep must be at rounding level (a stale
multi-rank allreduce once left the totals unsummed)."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("halo_mode", [0, 2])
def test_two_rank_bench_line(halo_mode):
    env = dict(os.environ, AMR_BENCH_HOST_COMM="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus", "2", "--steps", "3", "--warmup", "3",
           "--N", "1024", "--halo-mode", str(halo_mode), "--no-weno", "--no-amr", "--no-sweep-table",
           "--no-cpu-baseline"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["e2e"]["value"] > 0
    assert d["conservation_drift_per_step"] < 1e-12
    assert "TEST transport" in d["config"]["parallelism"]
