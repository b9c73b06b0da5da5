#!/usr/bin/env python
"""Benchmark of the B200 AMR compressible-Euler hot path (BASELINE.json metric:
"Euler cell-updates/sec per RK stage at 1/2/4/8 B200; achieved HBM GB/s vs peak").

    python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference] [--workload sweep|vortex|quadrant]

Default workload: BASELINE.json configs[4] (uniform-patch throughput sweep) at 4096^2 cells per GPU
(weak scaling, D5w), 32^2 patches, periodic, per-cell noise states from SplitMix64 seed 7, Central4
(Eq. 8/9) with SSP-RK3; dt fixed from step 0 (CFL 0.3).  A step = one full SSP-RK3 step (3 fused stage
launches plus the step's dt/Lambda work).  Before every timed step U^n is restored from a pristine copy
(a 537 MB device-to-device write that also flushes the 126 MB L2; outside the timed intervals), so every
timed step starts from the same positive state.  One JSON line is printed by rank 0.
Multi-GPU (torchrun): each rank owns a 4096^2 slab of a periodic (4096 N) x 4096 domain... see DESIGN.md s6.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import workloads as W  # noqa: E402


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d.get("hbm_gbs", 6650.0), "measured"
    return 6650.0, "fallback"


class Clocks:
    """nvidia-smi sampling of SM clocks and throttle reasons during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                f = [x.strip() for x in out.stdout.strip().split(",")]
                if len(f) >= 6:
                    self.samples.append(f)
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=6)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for s in self.samples for k in range(4) if s[2 + k].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def workload(args, world):
    if args.workload == "sweep":
        # D5w: 4096^2 cells per GPU, slabs stacked in y (weak scaling)
        cfg = W.sweep(N=args.N, n=args.n, scheme=args.scheme, Ny=args.N * world, seed=7)
        cfg["characteristic"] = args.characteristic
        cfg["check_positivity"] = 0
        name = (f"BASELINE configs[4] uniform-patch sweep, {args.N}x{args.N * world} cells "
                f"({args.N}^2 per GPU), {args.n}^2 patches, periodic, noise seed 7")
    elif args.workload == "vortex":
        cfg = W.vortex(N=1024, n=32)
        name = "BASELINE configs[1] isentropic vortex 1024^2, 32^2 patches"
    else:
        raise SystemExit(f"unknown workload {args.workload}")
    return cfg, name


def algorithmic_bytes_per_cell_stage():
    # stage 1 reads U^n (32 B) + writes 32 B; stages 2-3 read U^(s-1), U^n, write: 96 B
    return (64.0 + 96.0 + 96.0) / 3.0


def run_reference(args):
    """--impl reference: the CPU oracle as it stands, on a bounded sample of the same workload."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle as orc
    world = int(os.environ.get("WORLD_SIZE", "1"))
    cfg, name = workload(args, 1)
    # bounded sample: a 256^2 periodic piece of the same noise field (same per-cell work), K steps
    sub = dict(cfg, base=(256, 256), hi=(256 / 4096.0, 256 / 4096.0))
    o = orc.Oracle(sub)
    U0 = W.level0_state(sub)
    o.set_state(lambda l, P, Q: U0[Q, P])
    lam = o.lam()
    dt = args.cfl / lam
    t0 = time.perf_counter()
    steps = max(1, min(args.steps, 3))
    for _ in range(steps):
        o.set_state(lambda l, P, Q: U0[Q, P])
        try:
            o.step(dt=dt)
        except Exception:
            pass
    el = time.perf_counter() - t0
    v = 256 * 256 * 3 * steps / el
    line = {"impl": "reference", "metric": "Euler cell-updates/sec per RK stage", "value": v,
            "unit": "cell-updates/s", "n_gpus": world, "steps": steps, "warmup": 0, "ms_per_step": el / steps * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": name, "scheme": args.scheme},
            "cpu_baseline": {"value": v, "unit": "cell-updates/s", "cores": 1, "kind": "oracle",
                             "sample": f"256^2 periodic piece of the same noise field, {steps} SSP-RK3 steps"},
            "e2e": {"value": v, "unit": "cell-updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def cpu_baseline(args, cfg):
    import oracle as orc
    sub = dict(cfg, base=(256, 256), hi=(256 / 4096.0, 256 / 4096.0))
    o = orc.Oracle(sub)
    U0 = W.level0_state(sub)
    o.set_state(lambda l, P, Q: U0[Q, P])
    dt = args.cfl / o.lam()
    t0 = time.perf_counter()
    k = 0
    while True:
        o.set_state(lambda l, P, Q: U0[Q, P])
        try:
            o.step(dt=dt)
        except Exception:
            pass
        k += 1
        if time.perf_counter() - t0 > args.cpu_seconds or k >= 50:
            break
    el = time.perf_counter() - t0
    return {"value": 256 * 256 * 3 * k / el, "unit": "cell-updates/s", "cores": 1, "kind": "oracle",
            "sample": f"256^2 periodic piece of the same noise field, {k} SSP-RK3 steps, single thread"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="sweep", choices=["sweep", "vortex"])
    ap.add_argument("--scheme", default="central4", choices=["central4", "weno5"])
    ap.add_argument("--characteristic", type=int, default=1)
    ap.add_argument("--N", type=int, default=4096)
    ap.add_argument("--n", type=int, default=32)
    ap.add_argument("--cfl", type=float, default=0.3)
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-weno", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    from paper_2508_05020_b200 import build as B
    if rank == 0:
        B.build()
    if world > 1:
        dist.barrier()
    import paper_2508_05020_b200 as amr

    cfg, name = workload(args, world)
    stream = torch.cuda.Stream()   # the library launches on this stream; CUDA events are recorded on it
    hbm_peak, peak_kind = peaks()

    def measure(scheme, characteristic, steps, warmup, do_e2e):
        c = dict(cfg, scheme=scheme, characteristic=characteristic)
        mesh = amr.Mesh(c, stream=stream, **({} if world == 1 else {}))
        n = c["n"]
        U0h = W.level0_state(c).reshape(-1, 4, n, n)
        npatch = U0h.shape[0]
        mesh.set_state(U=U0h)
        pristine = mesh.get_state(as_dict=False)
        # device copy of the pristine state for restores between timed steps
        idx = np.arange(npatch, dtype=np.int32)
        _, lam = mesh.diagnostics()
        dt = args.cfl / lam
        U0d = torch.from_numpy(pristine).cuda()
        host_pinned = torch.from_numpy(pristine).pin_memory()
        torch.cuda.synchronize()

        def restore():
            # untimed: pristine device copy -> U^n (537 MB device-to-device; also flushes the 126 MB L2)
            mesh.set_state_device(U0d)

        for _ in range(warmup):
            restore()
            mesh.step(dt=dt, want_dt=False)
        torch.cuda.synchronize()
        mesh.reset_stats()
        mesh.set_kernel_timing(True)
        times = []
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        wall0 = time.perf_counter()
        with Clocks(local) as clk:
            for _ in range(steps):
                restore()
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                mesh.steps(1, dt=dt)
                e1.record(stream)
                e1.synchronize()
                times.append(e0.elapsed_time(e1))
        torch.cuda.synchronize()
        wall = time.perf_counter() - wall0
        if world > 1:
            dist.barrier()
        st = mesh.stats()
        mesh.set_kernel_timing(False)
        ms = sum(times)
        if world > 1:
            t = torch.tensor([ms], device="cuda", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        cells = st["leaf_cells"] * world
        value = cells * 3 * steps / (ms / 1e3)
        # roofline of the dominant kernel (the fused stage kernel), CUDA events on the launch stream
        stage_avg_ms = st["stage_ms"] / max(1, st["stage_timed"])
        bytes_per_launch = st["stage_bytes"] / max(1, st["stage_timed"])
        achieved = bytes_per_launch / (stage_avg_ms / 1e3) / 1e9
        res = {"value": value, "ms_per_step": ms / steps, "wall_s": wall, "stats": st, "clocks": clk.summary(),
               "stage_share": st["stage_ms"] / ms if ms > 0 else None,
               "roofline": {"bound": "hbm" if scheme == "central4" else "alu", "achieved": achieved,
                            "peak": hbm_peak, "unit": "GB/s", "frac": achieved / hbm_peak, "traffic": None,
                            "peak_kind": peak_kind,
                            "kernel": "stage_kernel (fused reconstruction+flux+divergence+RK)",
                            "algorithmic_bytes_per_cell_stage": algorithmic_bytes_per_cell_stage(),
                            "avg_launch_ms": stage_avg_ms},
               "gpu_launches": st["launches"]}
        if do_e2e:
            # end to end through the public API with host buffers: upload the state from pinned host memory,
            # K steps each reading dt_used back (D2H), download the final state -- all inside the timed region.
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            out = np.empty_like(pristine)
            e0.record(stream)
            mesh.set_state(U=host_pinned.numpy())
            for _ in range(steps):
                mesh.step(dt=dt, want_dt=True)
            mesh.L.amr_get_state(mesh.h, npatch, idx.ctypes.data_as(amr._I32), out.ctypes.data_as(amr._D))
            e1.record(stream)
            e1.synchronize()
            ems = e0.elapsed_time(e1)
            if world > 1:
                t = torch.tensor([ems], device="cuda", dtype=torch.float64)
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                ems = float(t.item())
            sb = pristine.nbytes
            res["e2e"] = {"value": cells * 3 * steps / (ems / 1e3), "unit": "cell-updates/s",
                          "h2d_bytes_per_step": sb / steps, "d2h_bytes_per_step": sb / steps + 8}
        mesh.close()
        del U0d
        return res

    main_res = measure(args.scheme, args.characteristic, args.steps, args.warmup, True)
    extra = {}
    if not args.no_weno and args.scheme == "central4":
        wr = measure("weno5", 1, max(3, args.steps // 2), 2, False)
        extra["weno5_char"] = {"value": wr["value"], "ms_per_step": wr["ms_per_step"], "roofline": wr["roofline"],
                               "positivity": "not held (noise input; see DESIGN.md s6)"}
    if rank == 0:
        line = {"metric": "Euler cell-updates/sec per RK stage", "value": main_res["value"], "unit": "cell-updates/s",
                "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": main_res["ms_per_step"],
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic",
                "config": {"workload": name, "scheme": args.scheme, "patch": args.n, "cfl_fixed_dt": args.cfl,
                           "parallelism": f"patch-partition x{world}" if world > 1 else "single GPU",
                           "l2": "inputs (3 x 537 MB buffers) larger than L2; U^n restored from a pristine copy "
                                 "between timed steps (untimed, also flushes L2)",
                           "positivity": "held for every timed step (check disabled in the timed region)"},
                "roofline": main_res["roofline"], "e2e": main_res.get("e2e"),
                "clocks": main_res["clocks"], "gpu_launches": main_res["gpu_launches"],
                "stage_kernel_share": main_res["stage_share"]}
        if not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(args, cfg)
        line.update(extra)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
