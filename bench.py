#!/usr/bin/env python
"""Benchmark of the B200 AMR compressible-Euler hot path (BASELINE.json metric:
"Euler cell-updates/sec per RK stage at 1/2/4/8 B200; achieved HBM GB/s vs peak").

    python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference] [--workload sweep|vortex]
    torchrun --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N ...

Headline workload: BASELINE.json configs[4] (uniform-patch throughput sweep) at 4096^2 cells PER GPU (weak
scaling: a 4096 x 4096N periodic domain, rank r owning one 4096^2 square through the Morton
root partition), 32^2 patches, per-cell noise states from SplitMix64 seed 7, Central4 (Eq. 8/9) + SSP-RK3,
dt fixed from step 0 (CFL 0.3).  A step = one full SSP-RK3 step through amr_steps (3 fused stage launches,
the dt/Lambda work and, for N > 1, 3 halo exchanges and the Lambda allreduce over NCCL).  Before every
timed step U^n is restored from a pristine device copy (537 MB per GPU, untimed; it also flushes the 126 MB
L2), so every timed step starts from the same positive state.  Rank 0 prints one JSON line with the
WENO5-characteristic stage throughput and the 3-level quadrant AMR step (BASELINE configs[2], regrid every
4 steps) as extra keys.
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

BYTES_PER_CELL_STAGE = (64.0 + 96.0 + 96.0) / 3.0   # U^n (+U^(s-1)) read, U^(s) written, fp64


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d.get("hbm_gbs", 6650.0), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def fp64_peak():
    """Sustained DFMA TFLOP/s measured by scripts/dfma_peak on this pool (profiles/dfma_peak.json), else the
    guide's unit-count estimate 148 SM x 64 DFMA/clk x 2 flops x 1.965 GHz."""
    p = os.path.join(ROOT, "profiles", "dfma_peak.json")
    if os.path.exists(p):
        return json.load(open(p))["fp64_dfma_tflops"], "measured (profiles/dfma_peak.json)"
    return 148 * 64 * 2 * 1.965e9 / 1e12, "derived (148 SM x 64 DFMA/clk x 2 x 1.965 GHz)"


def fp64_work(kernel, n=None):
    """fp64 SASS work per leaf cell-stage of a stage kernel (kernel "weno5_char" / "central4" at patch size n, whose
    launch configuration differs), counted by ncu on the current kernels (profiles/r2i_fp64_work.json, scripts/profile_round.sh)."""
    p = os.path.join(ROOT, "profiles", "r2i_fp64_work.json")
    d = json.load(open(p)) if os.path.exists(p) else {}
    nan = {"fp64_thread_inst_per_cell_stage": float("nan"), "flops_per_cell_stage": float("nan")}
    if n is not None and f"{kernel}_n{min(n, 32)}" in d:
        return d[f"{kernel}_n{min(n, 32)}"]
    return d.get(kernel, nan)


class Clocks:
    """SM clocks and throttle reasons sampled during the timed region: NVML polled every ~2 ms (the headline's
    timed region is ~11 ms, where nvidia-smi's ~100 ms cadence gave one sample), else nvidia-smi."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.samples = []
        self.source = "nvidia-smi"
        self._stop = threading.Event()
        self._nvml = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nvml = (pynvml, pynvml.nvmlDeviceGetHandleByIndex(index))
            self.source = "nvml"
        except Exception:
            self._nvml = None
        self._t = threading.Thread(target=self._run_nvml if self._nvml else self._run, daemon=True)

    def _run_nvml(self):
        nv, h = self._nvml
        bits = [nv.nvmlClocksEventReasonHwSlowdown, nv.nvmlClocksEventReasonHwThermalSlowdown,
                nv.nvmlClocksEventReasonSwThermalSlowdown, nv.nvmlClocksEventReasonSwPowerCap]
        try:
            mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        except Exception:
            mx = 0
        while not self._stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.samples.append([str(sm), str(mx)] + ["Active" if r & b else "Not Active" for b in bits])
            except Exception:
                pass
            self._stop.wait(0.002)

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
            self._stop.wait(0.1)

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
                "reasons": reasons, "samples": len(self.samples), "source": self.source,
                "sm_mhz_min": min(sm) if sm else None}


def sweep_cfg(args, world, scheme, characteristic=1):
    cfg = W.sweep(N=args.N, n=args.n, scheme=scheme, Ny=args.N * world, seed=7)
    cfg["characteristic"] = characteristic
    cfg["check_positivity"] = 0
    cfg["stage_kernel"] = args.stage_kernel
    cfg["halo_mode"] = args.halo_mode
    cfg["peer_map"] = args.peer_map
    name = (f"BASELINE configs[4] uniform-patch sweep: {args.N}x{args.N * world} cells ({args.N}^2 per GPU, "
            f"D5w weak scaling), {args.n}^2 patches, periodic, noise seed 7")
    return cfg, name


# --------------------------------------------------------------------------------------- reference arm
def host_cpu():
    """The host the oracle runs on: logical CPUs usable by this process and the lscpu model name."""
    model = None
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.lower().startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    try:
        usable = len(os.sched_getaffinity(0))
    except Exception:
        usable = os.cpu_count()
    return {"model": model, "logical_cpus": os.cpu_count(), "usable_cpus": usable}


def oracle_rate(cfg, cfl, seconds, threads=1, size=256, max_steps=100000, min_steps=1):
    """The CPU oracle as it stands (OpenMP over patches with `threads` threads; deterministic) on a size^2
    periodic piece of the same field (the same per-cell work).  Every step starts from the pristine piece; the
    restore (marshalling through ctypes) is outside the timed calls, so only amr-equivalent orc_step time counts.
    Returns (cell-updates/s per RK stage, steps, seconds timed)."""
    import oracle as orc
    orc.set_num_threads(threads)
    sub = dict(cfg, base=(size, size), hi=(size / 4096.0, size / 4096.0))
    o = orc.Oracle(sub)
    U0 = W.level0_state(sub)
    o.set_state(lambda l, P, Q: U0[Q, P])
    dt = cfl / o.lam()
    el, k = 0.0, 0
    while (el < seconds or k < min_steps) and k < max_steps:
        o.set_state(lambda l, P, Q: U0[Q, P])
        t0 = time.perf_counter()
        o.step(dt=dt)                  # check_positivity is 0 for the sweep: never raises
        el += time.perf_counter() - t0
        k += 1
    return size * size * 3 * k / el, k, el


def run_reference(args):
    """--impl reference: the CPU oracle (there is no installable reference implementation: the reference is a
    paper), timed on all of the host's cores, on this arm's workload: K timed steps after W warm-up steps, each an
    SSP-RK3 step of a 1024^2 periodic piece of the same noise field (the same per-cell work as the GPU's
    4096^2-per-GPU step, a bounded sample of it).  Under torchrun only rank 0 runs."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    world = int(os.environ.get("WORLD_SIZE", "1"))
    import oracle as orc
    orc.build()
    cpu = host_cpu()
    threads = cpu["usable_cpus"] or 1
    cfg, name = sweep_cfg(args, world, args.scheme)
    size = 1024
    oracle_rate(cfg, args.cfl, 0.0, threads=threads, size=size, max_steps=max(1, args.warmup), min_steps=args.warmup)
    v, k, el = oracle_rate(cfg, args.cfl, 0.0, threads=threads, size=size, max_steps=args.steps,
                           min_steps=args.steps)
    sample = (f"{size}^2 periodic piece of the same noise field per step, {k} timed SSP-RK3 steps after "
              f"{args.warmup} warm-up, OpenMP over patches with {threads} threads on {cpu['model']}")
    line = {"impl": "reference", "metric": "Euler cell-updates/sec per RK stage", "value": v,
            "unit": "cell-updates/s", "n_gpus": world, "steps": k, "warmup": args.warmup,
            "ms_per_step": el / k * 1e3,
            "ms_per_step_note": f"one SSP-RK3 step of the {size}^2 sample",
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": name, "scheme": args.scheme, "patch": args.n, "cfl_fixed_dt": args.cfl},
            "cpu_baseline": {"value": v, "unit": "cell-updates/s", "cores": threads, "kind": "oracle",
                             "sample": sample, "host": cpu},
            "e2e": {"value": v, "unit": "cell-updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------------------- our arm
class Ctx:
    def __init__(self):
        import torch
        import torch.distributed as dist
        self.torch, self.dist = torch, dist
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        # AMR_BENCH_HOST_COMM=1 (test only): every rank on GPU 0, a gloo process group and the library's host-
        # collective transport (comm_backend 2, CUDA IPC peer pools) -- exercises the N > 1 bench logic on one GPU;
        # its numbers are not multi-GPU numbers
        self.host_comm = os.environ.get("AMR_BENCH_HOST_COMM", "0") == "1"
        self.dev = 0 if self.host_comm else self.local
        torch.cuda.set_device(self.dev)
        if self.world > 1:
            if self.host_comm:
                dist.init_process_group("gloo")
            else:
                dist.init_process_group("nccl", device_id=torch.device("cuda", self.local))
        from paper_2508_05020_b200 import build as B
        # the library of this source tree (an mtime no-op when it is fresh); AMR_NO_BUILD=1 keeps a swapped-in prebuilt
        # library (A/B of two builds, scripts/ab_so.sh)
        if self.rank == 0 and os.environ.get("AMR_NO_BUILD", "0") != "1":
            B.build()
        self.barrier()
        import paper_2508_05020_b200 as amr
        self.amr = amr
        self.stream = torch.cuda.Stream()   # the library launches here; CUDA events are recorded here

    def barrier(self):
        if self.world > 1:
            self.dist.barrier()

    def max_over_ranks(self, x):
        if self.world == 1:
            return x
        t = self.torch.tensor([x], device="cpu" if self.host_comm else "cuda", dtype=self.torch.float64)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def min_over_ranks(self, x):
        return -self.max_over_ranks(-x)

    def sum_over_ranks(self, x):
        if self.world == 1:
            return x
        t = self.torch.tensor([float(x)], device="cpu" if self.host_comm else "cuda", dtype=self.torch.float64)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM)
        return float(t.item())

    def mesh(self, cfg):
        kw = {}
        if self.world > 1 and self.host_comm:
            kw = dict(world_size=self.world, rank=self.rank, comm_backend=2)
        elif self.world > 1:
            ids = [self.amr.nccl_unique_id() if self.rank == 0 else None]
            self.dist.broadcast_object_list(ids, src=0)
            kw = dict(world_size=self.world, rank=self.rank, comm_backend=0, comm_id=ids[0])
        return self.amr.Mesh(cfg, stream=self.stream, **kw)


def measure_sweep(X, args, cfg, steps, warmup, do_e2e):
    torch = X.torch
    mesh = X.mesh(cfg)
    n = cfg["n"]
    npx = cfg["base"][0] // n
    own = mesh.owned()
    q0, q1 = int(own[0]) // npx, int(own[-1]) // npx + 1
    assert np.array_equal(own, np.arange(q0 * npx, q1 * npx)), "expected one slab of patch rows per rank"
    U0 = W.level0_state(cfg, rows=(q0, q1)).reshape(-1, 4, n, n)
    mesh.set_state(U=U0, indices=own)
    _, lam = mesh.diagnostics()
    dt = args.cfl / lam
    U0d = torch.from_numpy(U0).cuda()
    pinned = torch.from_numpy(U0).pin_memory()
    torch.cuda.synchronize()

    def restore():   # untimed: pristine device copy -> U^n (537 MB / GPU; also flushes the L2)
        mesh.set_state_device(U0d, indices=own)

    for _ in range(warmup):
        restore()
        mesh.steps(1, dt=dt)
    torch.cuda.synchronize()
    mesh.reset_stats()
    mesh.set_kernel_timing(True)
    times = []
    X.barrier()
    torch.cuda.synchronize()
    wall0 = time.perf_counter()
    with Clocks(X.dev) as clk:
        for _ in range(steps):
            restore()
            X.barrier()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(X.stream)
            mesh.steps(1, dt=dt)
            e1.record(X.stream)
            e1.synchronize()
            times.append(e0.elapsed_time(e1))
    torch.cuda.synchronize()
    X.barrier()
    wall = time.perf_counter() - wall0
    st = mesh.stats()
    mesh.set_kernel_timing(False)
    tot1, _ = mesh.diagnostics()          # after the last timed step (which started from the pristine state)
    Uf = torch.empty_like(U0d)
    mesh.get_state_device(Uf, indices=own)
    torch.cuda.synchronize()
    rho, E = Uf[:, 0], Uf[:, 3]
    pres = (cfg.get("gamma", 1.4) - 1.0) * (E - 0.5 * (Uf[:, 1] ** 2 + Uf[:, 2] ** 2) / rho)
    pos = {"min_rho": X.min_over_ranks(float(rho.min())), "min_p": X.min_over_ranks(float(pres.min()))}
    del Uf, rho, E, pres
    restore()
    tot0, _ = mesh.diagnostics()
    scale = max(abs(float(x)) for x in tot0)
    drift = max(abs(float(a) - float(b)) for a, b in zip(tot1, tot0)) / scale
    ms = X.max_over_ranks(sum(times))
    cells = X.sum_over_ranks(st["leaf_cells"])
    value = cells * 3 * steps / (ms / 1e3)
    stage_avg_ms = st["stage_ms"] / max(1, st["stage_timed"])
    bytes_per_launch = st["stage_bytes"] / max(1, st["stage_timed"])
    achieved = bytes_per_launch / (stage_avg_ms / 1e3) / 1e9
    res = {"value": value, "ms_per_step": ms / steps, "wall_s": wall, "stats": st, "clocks": clk.summary(),
           "stage_share": st["stage_ms"] / sum(times) if times else None, "achieved_gbs": achieved,
           "stage_avg_ms": stage_avg_ms, "cells_per_launch": st["stage_cells"] / max(1, st["stage_timed"]),
           "gpu_launches": st["launches"], "conservation_drift_per_step": drift, "positivity": pos}
    if do_e2e:
        # end to end through the public API with host buffers: the state uploaded from pinned host memory,
        # K steps each reading dt_used back (D2H), the final state downloaded -- all inside the timed region.
        out = torch.empty(U0.shape, dtype=torch.float64).pin_memory().numpy()   # the download's host buffer
        torch.cuda.synchronize()
        X.barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(X.stream)
        mesh.set_state(U=pinned.numpy(), indices=own)
        for _ in range(steps):
            mesh.step(dt=dt, want_dt=True)
        mesh.get_state(as_dict=False, indices=own, out=out)
        e1.record(X.stream)
        e1.synchronize()
        ems = X.max_over_ranks(e0.elapsed_time(e1))
        sb = U0.nbytes
        res["e2e"] = {"value": cells * 3 * steps / (ems / 1e3), "unit": "cell-updates/s",
                      "h2d_bytes_per_step": sb / steps, "d2h_bytes_per_step": sb / steps + 8,
                      "includes": "amr_set_state from pinned host, K x amr_step(dt, &dt_used), amr_get_state into "
                                  "pinned host"}
    mesh.close()
    return res


def measure_sweep_table(X, args, hbm_peak):
    """BASELINE configs[4] as stated: totals 4096^2, 8192^2, 16384^2 x patches 8/16/32/64 (Central4, one GPU).
    The 4096^2 noise field of each patch size is generated once and tiled periodically on the device for the
    larger totals (a valid periodic state with the same statistics); per configuration the fused stage kernel's
    CUDA-event time over 3 steps after 1 warm-up step, each step from the pristine state."""
    torch = X.torch
    rows = []
    fpk_inst = 148 * 64 * 1.965e9
    for n in (8, 16, 32, 64):
        small = W.sweep(N=4096, n=n, scheme="central4", seed=7)
        U0 = torch.from_numpy(W.level0_state(small)).cuda()
        runs = [(N, "central4", 1) for N in (4096, 8192, 16384)] + [(4096, "weno5", 1), (4096, "weno5", 0)]
        for N, scheme, char in runs:
            r = N // 4096
            cfg = W.sweep(N=N, n=n, scheme=scheme, seed=7)
            cfg.update(check_positivity=0, stage_kernel=args.stage_kernel, characteristic=char)
            mesh = X.mesh(cfg)
            Ut = U0.repeat(r, r, 1, 1, 1).reshape(-1, 4, n, n).contiguous()
            torch.cuda.synchronize()   # Ut is written on torch's stream; the library reads it on its own
            idx = np.arange(Ut.shape[0], dtype=np.int32)
            mesh.set_state_device(Ut, indices=idx)
            _, lam = mesh.diagnostics()
            dt = args.cfl / lam
            mesh.steps(1, dt=dt)
            mesh.reset_stats()
            mesh.set_kernel_timing(True)
            for _ in range(3):
                mesh.set_state_device(Ut, indices=idx)
                mesh.steps(1, dt=dt)
            torch.cuda.synchronize()
            st = mesh.stats()
            mesh.set_kernel_timing(False)
            mesh.close()
            del Ut
            ms = st["stage_ms"] / max(1, st["stage_timed"])
            cells = st["stage_cells"] / max(1, st["stage_timed"])
            gbs = st["stage_bytes"] / max(1, st["stage_timed"]) / (ms / 1e3) / 1e9
            row = {"N": N, "n": n, "scheme": scheme if scheme == "central4" else ("weno5_char" if char else "weno5_comp"),
                   "stage_ms": ms, "cell_updates_per_s": cells / (ms / 1e3), "hbm_gbs": gbs, "hbm_frac": gbs / hbm_peak}
            if scheme == "weno5" and char:   # fp64-issue bound: SASS instruction count of the WENO5-char kernel
                row["fp64_issue_frac"] = fp64_work("weno5_char", n)["fp64_thread_inst_per_cell_stage"] * row["cell_updates_per_s"] / fpk_inst
            rows.append(row)
        del U0
        torch.cuda.empty_cache()
    return rows


def measure_quadrant(X, args, use_graphs=0):
    """BASELINE configs[2]: quadrant Riemann problem, 512^2 base, 3 levels, WENO5-char, regrid every 4 steps.
    Timed: K steps including the regrids (flags, Alg. 1/2, prolongation, migration) inside the region.
    use_graphs = 1: each step is a CUDA-graph replay (re-captured after each regrid)."""
    cfg = dict(W.quadrant(N=512, n=16, levels=3, seed=1), use_graphs=use_graphs if X.world == 1 else 0)
    return measure_amr(X, cfg, "BASELINE configs[2] quadrant AMR, 512^2 base, 3 levels, 16^2 patches, WENO5-char, "
                               "8 CFL-0.5 steps with 2 regrids inside the timed region")


def measure_amr(X, cfg, workload, windows=3):
    """An AMR config: init protocol (A28), 8 untimed steps with two regrids, then `windows` timed windows of 8
    CFL-0.5 steps with a regrid every 4 steps inside each (CUDA events on the library stream; the host regrid
    work is on the timeline).  The 4 steps between regrids are one amr_steps call (queued without a host round trip
    per step; positivity is still checked on the device and reported at the regrid's synchronisation).  The mesh
    keeps evolving across windows; the median window is reported (a single 8-step window is exposed to host
    hiccups), all windows are listed.  Also the simulated time advanced per second (amr_stats.sim_time)."""
    torch = X.torch
    mesh = X.mesh(cfg)
    fn = lambda l, P, Q: W.patch_state(cfg, l, P, Q)   # noqa: E731
    mesh.set_state(fn)
    for _ in range(cfg["levels"] - 1):
        mesh.regrid()
        mesh.set_state(fn)
    for _ in range(2):                 # warm-up incl. two regrids (first launches load the regrid kernels)
        mesh.steps(4, cfl=0.5)
        mesh.regrid()
    torch.cuda.synchronize()
    X.barrier()
    steps = 8
    res = []
    for _ in range(windows):
        leaf_cells = 0
        t_sim0 = mesh.stats()["sim_time"]
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        X.barrier()
        e0.record(X.stream)
        rg = 0.0
        for _ in range(steps // 4):
            leaf_cells += 4 * mesh.stats()["leaf_cells"]
            mesh.steps(4, cfl=0.5)
            mesh.sync()                # (the regrid synchronises anyway: its own time is measured from here)
            t0 = time.perf_counter()
            mesh.regrid()
            rg += time.perf_counter() - t0
        e1.record(X.stream)
        e1.synchronize()
        sim_t = mesh.stats()["sim_time"] - t_sim0
        ms = X.max_over_ranks(e0.elapsed_time(e1))
        res.append((ms, X.sum_over_ranks(leaf_cells), sim_t, X.max_over_ranks(rg * 1e3)))
    st = mesh.stats()
    mesh.close()
    ms, cells, sim_t, rg_ms = sorted(res)[len(res) // 2]
    out = {"value": cells * 3 / (ms / 1e3), "ms_per_step": ms / steps, "leaves": st["leaves"],
           "patches": st["patches"], "leaf_cells_last": st["leaf_cells"], "workload": workload,
           "simulated_time_per_s": sim_t / (ms / 1e3),
           "windows_ms_per_step": [r[0] / steps for r in res], "reported": "median window",
           "regrid_ms_per_call": rg_ms / (steps // 4),
           "step_ms_without_regrid": (ms - rg_ms) / steps}
    if cfg.get("subcycle"):
        out["value_note"] = "leaf cell-updates counted once per level-0 step (finer levels update 2^l times)"
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--scheme", default="central4", choices=["central4", "weno5"])
    ap.add_argument("--characteristic", type=int, default=1)
    ap.add_argument("--N", type=int, default=4096)
    ap.add_argument("--n", type=int, default=32)
    ap.add_argument("--cfl", type=float, default=0.3)
    ap.add_argument("--stage-kernel", type=int, default=0, help="amr_config.stage_kernel (0 default, 1 per-tile)")
    ap.add_argument("--peer-map", type=int, default=0, choices=[0, 1],
                    help="halo_mode 1/2 peer mapping: 0 CUDA IPC, 1 NCCL symmetric windows (ncclMemAlloc pool)")
    ap.add_argument("--halo-mode", type=int, default=0, choices=[0, 1, 2],
                    help="N > 1 halo exchange: 0 pack + NCCL send/recv + unpack, 1 peer pull over CUDA IPC, "
                         "2 remote face strips loaded by the stage kernel from the peers' pools (NEXT #3)")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-weno", action="store_true")
    ap.add_argument("--no-amr", action="store_true")
    ap.add_argument("--no-sweep-table", action="store_true",
                    help="skip the configs[4] size x patch-size table (single GPU only)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    X = Ctx()
    hbm_peak, hbm_kind = peaks()
    cfg, name = sweep_cfg(args, X.world, args.scheme, args.characteristic)
    main_res = measure_sweep(X, args, cfg, args.steps, args.warmup, True)
    extra = {}
    if not args.no_weno and args.scheme == "central4":
        wcfg, _ = sweep_cfg(args, X.world, "weno5", 1)
        wr = measure_sweep(X, args, wcfg, max(3, args.steps // 2), 2, False)
        fpk, fpk_kind = fp64_peak()
        work = fp64_work("weno5_char", args.n)
        rate = wr["cells_per_launch"] / (wr["stage_avg_ms"] / 1e3)          # cell-stages/s of the stage kernel
        inst_peak = 148 * 64 * 1.965e9 / 1e12                                  # T fp64 thread-inst/s (unit counts)
        extra["weno5_char"] = {
            "value": wr["value"], "unit": "cell-updates/s", "ms_per_step": wr["ms_per_step"],
            "roofline": {"bound": "alu", "unit": "T fp64 inst/s",
                         "achieved": work["fp64_thread_inst_per_cell_stage"] * rate / 1e12, "peak": inst_peak,
                         "frac": work["fp64_thread_inst_per_cell_stage"] * rate / 1e12 / inst_peak,
                         "peak_kind": "derived: 148 SM x 64 fp64 lanes x 1.965 GHz (DADD/DMUL/DFMA issue one each)",
                         "achieved_tflops": work["flops_per_cell_stage"] * rate / 1e12, "fp64_peak_tflops": fpk,
                         "fp64_peak_kind": fpk_kind, "work_per_cell_stage": work,
                         "achieved_hbm_gbs": wr["achieved_gbs"], "hbm_frac": wr["achieved_gbs"] / hbm_peak,
                         "stage_avg_ms": wr["stage_avg_ms"]},
            "positivity": "not held: WENO5-char reconstruction of white noise yields a few non-physical face "
                          "states (DESIGN.md s6); throughput config only"}
    if not args.no_amr:
        extra["quadrant_amr"] = measure_quadrant(X, args)
        G = X.world   # D4w: G mirrored copies of configs[3] stacked in y, one per GPU (weak scaling; G = 1: configs[3])
        extra["shock_bubble_amr"] = measure_amr(
            # slot capacity 100 k per copy (the problem keeps ~16 k active patches per copy); the default (every root
            # refined to the finest level, 5.6 M slots at G = 8) would take ~150 GB of pool per GPU
            X, W.shock_bubble(G=G, max_patches=100_000 * G), f"BASELINE configs[3] shock-bubble AMR{' (D4w weak scaling, %d copies)' % G if G > 1 else ''}, "
                                    f"2048x{1024 * G} base, 4 levels, 16^2 patches, WENO5-char, reflective walls, 8 CFL-0.5 "
                                    "steps with 2 regrids inside the timed region")
        if X.world == 1:   # NEXT #4: the same problem with Berger-Colella subcycling (level-0 steps)
            extra["shock_bubble_amr_subcycled"] = measure_amr(
                X, dict(W.shock_bubble(), subcycle=1),
                "configs[3] with time subcycling: 8 level-0 steps (each = 8 finest-level steps), 2 regrids")
    if not args.no_sweep_table and X.world == 1:
        extra["sweep_table"] = {"workload": "BASELINE configs[4]: stage kernel per total size and patch size (Central4 at "
                                            "4096^2..16384^2; WENO5 char / comp at 4096^2; fp64_issue_frac from each "
                                            "WENO5-char kernel's own SASS fp64 count, profiles/r2i_fp64_work.json)",
                                "rows": measure_sweep_table(X, args, hbm_peak)}
    if "sweep_table" in extra:   # the largest single-GPU configs[4] row beside the 4096^2-per-GPU headline
        big = [r for r in extra["sweep_table"]["rows"] if r["N"] == 16384 and r["n"] == args.n and r["scheme"] == args.scheme]
        if big:
            extra["largest_single_gpu"] = dict(big[0], workload="BASELINE configs[4] at its largest single-GPU size: "
                                                                 f"16384^2 cells, {args.n}^2 patches (stage kernel only)")
    if X.rank == 0:
        rf = {"bound": "hbm", "achieved": main_res["achieved_gbs"], "peak": hbm_peak, "unit": "GB/s",
              "frac": main_res["achieved_gbs"] / hbm_peak, "traffic": None, "peak_kind": hbm_kind,
              "kernel": ({8: "stage_c4_group_kernel<8>", 16: "stage_c4_group_kernel<16>"}.get(args.n, f"stage_c4_tma_kernel<{args.n}>")
                         if args.scheme == "central4" and args.stage_kernel == 0 else "stage kernel variant %d" % args.stage_kernel)
                        + " (TMA halo + cons->prim + Central4 flux + Eq. 9 divergence + SSP-RK3 update, one launch per stage)",
              "algorithmic_bytes_per_cell_stage": BYTES_PER_CELL_STAGE,
              "cells_per_launch": main_res["cells_per_launch"], "avg_launch_ms": main_res["stage_avg_ms"]}
        tf = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(tf):
            t = json.load(open(tf))
            rf["traffic"] = t.get("central4_bytes_per_launch")
            rf["traffic_note"] = t.get("note")
        line = {"metric": "Euler cell-updates/sec per RK stage", "value": main_res["value"], "unit": "cell-updates/s",
                "n_gpus": X.world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": main_res["ms_per_step"],
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (SplitMix64 noise, BASELINE configs[4] distributions)",
                "config": {"workload": name, "scheme": args.scheme, "patch": args.n, "cfl_fixed_dt": args.cfl,
                           "parallelism": (f"Morton root partition x{X.world}, " + (["NCCL halo exchange", "peer-pull halo (CUDA IPC, NVLink)", "remote strips read by the stage kernel (CUDA IPC, NVLink)"][args.halo_mode])
                                            + (" -- TEST transport: host collectives, all ranks on GPU 0" if X.host_comm else "")) if X.world > 1
                           else "single GPU",
                           "l2": "inputs larger than L2 (3 x 537 MB buffers per GPU); U^n restored from a pristine "
                                 "device copy between timed steps (untimed; also flushes L2)",
                           "positivity": "every timed step starts from the pristine state; minimum density and "
                                         "pressure after a step in the line's positivity key"},
                "roofline": rf, "e2e": main_res["e2e"], "clocks": main_res["clocks"],
                "gpu_launches": main_res["gpu_launches"], "stage_kernel_share": main_res["stage_share"],
                "conservation_drift_per_step": main_res["conservation_drift_per_step"],
                "positivity": main_res["positivity"]}
        if not args.no_cpu_baseline:
            cpu = host_cpu()
            nt = cpu["usable_cpus"] or 1
            v1, k1, el1 = oracle_rate(cfg, args.cfl, args.cpu_seconds / 2, threads=1, size=256)
            vn, kn, eln = oracle_rate(cfg, args.cfl, args.cpu_seconds / 2, threads=nt, size=1024)
            line["cpu_baseline"] = {
                "value": vn, "unit": "cell-updates/s", "cores": nt, "kind": "oracle",
                "sample": f"1024^2 periodic piece of the same noise field, {kn} SSP-RK3 steps ({eln:.1f} s timed), "
                          f"OpenMP over patches, {nt} threads",
                "host": cpu,
                "single_thread": {"value": v1, "cores": 1,
                                  "sample": f"256^2 piece, {k1} steps ({el1:.1f} s timed), 1 thread"}}
        line.update(extra)
        print(json.dumps(line), flush=True)
    if X.world > 1:
        X.dist.destroy_process_group()


if __name__ == "__main__":
    main()
