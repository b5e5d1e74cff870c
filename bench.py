#!/usr/bin/env python
"""Benchmark of the SIP hot path (BASELINE.json metric: SIP inner-iteration
MLUP/s and achieved HBM GB/s vs peak).

A "step" is one solve of the hot path over one synthetic system: `iters`
SIP inner iterations (residual + forward substitution K2, backward
substitution K3, face-halo exchange for multi-block) on the configuration's
grid.  MLUP/s = cells x iterations / time.

    python bench.py                      # N=1: config 1 (256^3, fp64 headline + fp32),
                                         #      configs 2, 3, 4 as sub-objects
    python bench.py --gpus N             # N>1: spawns N ranks (torchrun), BASELINE config 3
                                         #      (2x2x2 blocks of 128^3 per GPU, weak scaling)
    python bench.py --gpus N --config 4  # strong scaling: 1024x512x512 in 128 blocks, fp32
    python bench.py --impl reference     # reference arm: CPU SIP (oracle port) on host cores

value: device-resident throughput (inputs in HBM, CUDA events on the
library's launch stream, max over ranks).  e2e: the same metric through the
reference-facing call (sip_set_source + sip_solve with pinned host Field3
buffers: H2D of su and phi, D2H of phi and the norm history inside the
timed region).  roofline: dominant kernel (K2 forward) -- algorithmic bytes
per launch (14 of the 20 array touches per cell) over its
CUDA-event duration, against MEASURED_PEAKS.json's HBM copy bandwidth.
efficiency (N>1): Eq. 1 of the reference's perf report (perf.cpp:97-130),
eps = T_s / (N * T_p(N)), with T_s the 1-GPU time of the whole job measured
by rank 0 in the same run (weak scaling: N x the 1-GPU time of one GPU's share).
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# algorithmic array touches per lattice update
TOUCH_FWD, TOUCH_BWD = 14, 6

CONFIGS = {
    0: dict(workload="config0: 64^3 single block, 7-point SIP", g=(64, 64, 64), p=(1, 1, 1),
            kind=0, iters=20, prec=("f64",)),
    1: dict(workload="config1: 256^3 single block, 7-point SIP", g=(256, 256, 256), p=(1, 1, 1),
            kind=0, iters=50, prec=("f64", "f32")),
    2: dict(workload="config2: 512x256x128 anisotropic convection-diffusion block", g=(512, 256, 128),
            p=(1, 1, 1), kind=2, iters=100, prec=("f32",)),
    3: dict(workload="config3: 8 blocks of 128^3 per GPU (2x2x2 per GPU), block-Jacobi SIP",
            g=None, p=None, kind=0, iters=50, prec=("f64",)),
    4: dict(workload="config4: 1024x512x512 in 128^3 blocks (128 blocks), block-Jacobi SIP",
            g=(1024, 512, 512), p=(8, 4, 4), kind=0, iters=100, prec=("f32",)),
    # weak scaling of the headline workload: one config-1 block (256^3) per GPU,
    # GPUs in a block lattice, face halos exchanged every iteration (at N = 1
    # this is exactly config 1)
    5: dict(workload="config1xN: one 256^3 block per GPU (GPU lattice), block-Jacobi SIP, face halos",
            g=None, p=None, kind=0, iters=50, prec=("f64",)),
}
GPU_LATTICE = {1: (1, 1, 1), 2: (2, 1, 1), 4: (2, 2, 1), 8: (2, 2, 2)}


def load_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """SM clocks / throttle reasons sampled during the timed region: through
    NVML every 10 ms (the GPU matched by PCI bus id), else nvidia-smi (~0.1 s
    per query)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    # NVML clock-event reason bits, in the order of the names below
    BITS = (0x8, 0x40, 0x20, 0x4)  # hw_slowdown, hw_thermal, sw_thermal, sw_power_cap

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.source = "nvidia-smi"
        self._stop = threading.Event()
        self._nvml = None
        try:
            import pynvml
            import torch

            pynvml.nvmlInit()
            h = None
            try:
                pr = torch.cuda.get_device_properties(index)
                bus = f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
                h = pynvml.nvmlDeviceGetHandleByPciBusId(bus)
            except Exception:
                h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self._nvml = (pynvml, h)
            self.source = "nvml"
        except Exception:
            self._nvml = None
        self._t = threading.Thread(target=self._run, daemon=True)

    def _sample_nvml(self):
        nv, h = self._nvml
        sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        get = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            nv.nvmlDeviceGetCurrentClocksThrottleReasons
        r = get(h)
        return [str(sm), str(mx)] + ["Active" if r & b else "Not Active" for b in self.BITS]

    def _run(self):
        while not self._stop.is_set():
            try:
                if self._nvml:
                    self.samples.append(self._sample_nvml())
                else:
                    out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits"], capture_output=True,
                                         text=True, timeout=5).stdout.strip()
                    if out:
                        self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.01 if self._nvml else 0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["clock sampling unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 2 + i and s[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples), "source": self.source}


# ---------------------------------------------------------------- CPU reference
def cpu_reference(cfg_id: int, seconds: float = 12.0):
    """The reference's algorithm on the host with all the host threads it can
    use: the oracle port's sweep pipelined over j-slabs (one slab per core;
    phi bitwise equal to the serial sweep, tests/test_oracle.py).  Bounded
    sample: iterations of the config's grid until ~`seconds` of sweep time."""
    from oracle import oracle as O

    ncores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)

    c = CONFIGS[cfg_id]
    if cfg_id in (3, 4):
        dims = (128, 128, 128)  # one block of the multi-block configs
        sample_desc = "one 128^3 block of the config, fp64 sweeps"
    elif cfg_id == 5:
        dims = (256, 256, 256)  # one block (= one GPU's share) of the weak-scaling lattice
        sample_desc = "one 256^3 block (one GPU's share) of the config"
    else:
        dims = c["g"]
        sample_desc = f"{dims[0]}x{dims[1]}x{dims[2]} block"
    A = O.generate(c["kind"], 1303 + cfg_id, dims, dims)
    F = O.factor(A, 0.92)
    prec = c["prec"][0]
    if prec == "f32":
        A = {n: v.astype(np.float32) for n, v in A.items()}
        F = {n: v.astype(np.float32) for n, v in F.items()}
        phi = O.field(*dims, dtype=np.float32)
    else:
        phi = O.field(*dims)
    work = np.zeros_like(phi)
    cells = dims[0] * dims[1] * dims[2]
    n, t = 0, 0.0
    while t < seconds and n < 20 * c["iters"]:
        t0 = time.perf_counter()
        O.sweep_pipe(A, F, phi, ncores, work)
        t += time.perf_counter() - t0
        n += 1
    return {"value": cells * n / t / 1e6, "unit": "MLUP/s", "cores": ncores, "kind": "port",
            "sample": f"{sample_desc}, {prec}, {n} SIP inner iterations ({t:.1f} s), "
                      f"C oracle (-O3 -ffp-contract=off) pipelined over {ncores} host threads"}


# ---------------------------------------------------------------- GPU arm
def make_solver(cfg_id, prec, rank, world, device, nccl_id=None):
    import paper_1303_4538_b200 as sip

    c = CONFIGS[cfg_id]
    if cfg_id == 3:
        lx, ly, lz = GPU_LATTICE.get(world, (world, 1, 1))
        g = (256 * lx, 256 * ly, 256 * lz)
        p = (2 * lx, 2 * ly, 2 * lz)
    elif cfg_id == 5:
        lx, ly, lz = GPU_LATTICE.get(world, (world, 1, 1))
        g = (256 * lx, 256 * ly, 256 * lz)
        p = (lx, ly, lz)
    else:
        g, p = c["g"], c["p"]
    s = sip.Solver(None, prec, device, lattice=(g, p), rank=rank, nranks=world, nccl_id=nccl_id)
    s._g = g
    return s, g, p


def config_keys(cfg_id, world):
    """The `config` object of both arms (identical keys, so the two lines
    describe the same workload)."""
    c = CONFIGS[cfg_id]
    if cfg_id in (3, 5):
        lx, ly, lz = GPU_LATTICE.get(world, (world, 1, 1))
        g = (256 * lx, 256 * ly, 256 * lz)
        p = (2 * lx, 2 * ly, 2 * lz) if cfg_id == 3 else (lx, ly, lz)
    else:
        g, p = c["g"], c["p"]
    return {"workload": c["workload"], "grid": list(g), "blocks": list(p),
            "iters_per_step": c["iters"], "alpha": 0.92,
            "l2": "inputs larger than L2 (working set >> 126 MB)"}


def measure(cfg_id, prec, rank, world, dist, stream, steps, warmup, e2e_reps=0):
    """One configuration / precision on this rank's GPU(s): device-resident
    throughput (max over ranks), the per-kernel roofline pass and, if asked,
    the e2e call."""
    import torch

    import paper_1303_4538_b200 as sip

    c = CONFIGS[cfg_id]
    peak, peak_src = load_peak()
    nccl_id = None
    if world > 1:  # a fresh ncclUniqueId per communicator
        obj = [sip.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    s, g, p = make_solver(cfg_id, prec, rank, world, torch.cuda.current_device(), nccl_id)
    s.set_stream(stream.cuda_stream)
    seed = 1303 + (1 if cfg_id == 5 else cfg_id)
    s.generate(c["kind"], seed)
    s.factor(0.92)
    phis = [sip.field(*d) for (_, d, _) in s.blocks]  # resident phi0 = 0
    s.load_phi(phis)
    cells_local = sum(d[0] * d[1] * d[2] for (_, d, _) in s.blocks)
    cells_total = g[0] * g[1] * g[2]
    iters = c["iters"]

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(warmup):
        s.iterate(iters)
    barrier()
    l0 = s.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(torch.cuda.current_device()) as clk:
        ev0.record(stream)
        for _ in range(steps):
            s.iterate(iters)
        ev1.record(stream)
        barrier()
    ms = ev0.elapsed_time(ev1)
    launches = s.launch_count() - l0
    if dist is not None:
        t = torch.tensor([ms], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / steps
    mlups = cells_total * iters * steps / (ms / 1e3) / 1e6
    # norms of the run, read once after the timed region (sanity)
    nrm = s.read_norms(0, min(iters, 3))

    # per-kernel CUDA-event pass (same stream) for the roofline
    s.set_profiling(True)
    s.iterate(iters)
    prof = s.profile()
    s.set_profiling(False)
    esz = 8 if prec == "f64" else 4
    fwd_launch_ms = prof["fwd_ms"] / iters
    bwd_launch_ms = prof["bwd_ms"] / iters
    fwd_bytes = cells_local * TOUCH_FWD * esz
    bwd_bytes = cells_local * TOUCH_BWD * esz
    achieved = fwd_bytes / (fwd_launch_ms / 1e3) / 1e9
    bwd_achieved = bwd_bytes / (bwd_launch_ms / 1e3) / 1e9
    step_gbs = cells_local * (TOUCH_FWD + TOUCH_BWD) * esz * iters / (ms_step / 1e3) / 1e9
    e2e = run_e2e(s, c, cfg_id, prec, e2e_reps, dist, stream) if e2e_reps else None
    r = dict(
        value=mlups, ms=ms_step, launches=launches, clocks=clk.summary(), e2e=e2e,
        roofline={"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                  "frac": achieved / peak, "traffic": load_traffic(cfg_id, prec),
                  "kernel": "k_forward (K2)", "peak_source": peak_src,
                  "alg_bytes_per_launch": fwd_bytes, "launch_ms": fwd_launch_ms},
        k3={"kernel": "k_backward (K3)", "achieved": bwd_achieved, "frac": bwd_achieved / peak,
            "launch_ms": bwd_launch_ms, "alg_bytes_per_launch": bwd_bytes},
        step_gbs=step_gbs, step_frac=step_gbs / peak, halo_ms=prof["halo_ms"] / iters,
        kernel_ms_per_iter=(prof["fwd_ms"] + prof["bwd_ms"] + prof["halo_ms"]) / iters,
        first_norms=[float(x) for x in nrm], geometry=s.geometry(), cells_total=cells_total,
        cells_local=cells_local, g=g, p=p)
    s.close()
    return r


def summary(r, cfg_id, prec):
    """Sub-object of one extra configuration in the N=1 line."""
    return {"workload": CONFIGS[cfg_id]["workload"], "dtype": prec, "value": r["value"],
            "unit": "MLUP/s", "ms_per_step": r["ms"], "iters_per_step": CONFIGS[cfg_id]["iters"],
            "roofline_frac_k2": r["roofline"]["frac"], "roofline_frac_k3": r["k3"]["frac"],
            "k2_launch_ms": r["roofline"]["launch_ms"], "k3_launch_ms": r["k3"]["launch_ms"],
            "halo_ms_per_iter": r["halo_ms"], "achieved_frac_step": r["step_frac"],
            "gpu_launches": r["launches"], "clocks": r["clocks"]}


def run_e2e(s, c, cfg_id, prec, reps, dist, stream):
    import torch

    import paper_1303_4538_b200 as sip

    iters = c["iters"]
    # pinned host Field3 buffers (torch pin_memory), one per local block
    def pinned(d):
        t = torch.zeros((d[2] + 2, d[1] + 2, d[0] + 2), dtype=torch.float64).pin_memory()
        return t, t.numpy()

    phis = [pinned(d) for (_, d, _) in s.blocks]
    qs = []
    for (bid, d, o) in s.blocks:
        t, a = pinned(d)
        gen = sip.generate_host(c["kind"], 1303 + cfg_id + 17 + bid, d, s._g, o)
        a[...] = gen["Q"]
        qs.append((t, a))
    norms = np.zeros(iters)
    L = sip.lib()
    dp = ctypes.POINTER(ctypes.c_double)
    arr = (dp * len(phis))(*[p[1].ctypes.data_as(dp) for p in phis])
    used = ctypes.c_int()
    G = sum(p[1].size for p in phis)
    h2d = 2 * G * 8
    d2h = G * 8 + iters * 8

    qp = [a.ctypes.data_as(dp) for (t, a) in qs]
    nrm = [np.zeros(iters), np.zeros(iters)]
    pipelined = dist is None  # sip_solve_async is single-rank

    def run(reps):
        # every step: H2D of its inputs (Q and phi0 = the previous step's
        # result, a warm start; every step still runs all `iters` iterations,
        # target 0) from pinned host memory, the solve, D2H of phi and norms.
        # Single rank: pipelined -- the next step's Q is uploaded on the copy
        # stream while this step's solve runs (sip_set_source_async)
        if pipelined:
            # two steps in flight: step r+1's Q and phi0 uploads overlap step
            # r's solve and its phi download (phi0 = step r's result, uploaded
            # chunk by chunk as it arrives)
            def enqueue(r):
                for lb in range(len(qs)):
                    assert L.sip_set_source_async(s.handle, lb, qp[lb]) == 0
                st = L.sip_solve_async(s.handle, arr, iters, nrm[r % 2].ctypes.data_as(dp))
                assert st == 0, L.sip_last_error(s.handle)

            enqueue(0)
            for r in range(reps):
                if r + 1 < reps:
                    enqueue(r + 1)
                assert L.sip_wait_async(s.handle) == 0  # step r complete: phi and norms on the host
            return
        for _ in range(reps):
            for lb in range(len(qs)):
                assert L.sip_set_source(s.handle, lb, qp[lb]) == 0
            st = L.sip_solve(s.handle, arr, iters, ctypes.c_double(0.0), norms.ctypes.data_as(dp),
                             ctypes.byref(used))
            assert st == 0, L.sip_last_error(s.handle)

    run(1)  # warm
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    run(reps)
    torch.cuda.synchronize()
    el = time.perf_counter() - t0
    if dist is not None:
        t = torch.tensor([el], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        el = float(t.item())
    cells_total = s._g[0] * s._g[1] * s._g[2]
    return {"value": cells_total * iters * reps / el / 1e6, "unit": "MLUP/s",
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "ms_per_step": el / reps * 1e3, "steps": reps,
            "call": ("sip_set_source_async + sip_solve_async, two steps in flight (next step's Q and phi0 "
                     "uploads overlap this step's solve and phi download) + sip_wait_async"
                     if pipelined else "sip_set_source + sip_solve") +
                    " (pinned host Field3 buffers, phi0 = previous result)"}


def load_traffic(cfg_id, prec):
    """ncu dram bytes per launch of K2, from profiles/ncu_traffic.json if a
    capture of this config/precision was committed."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d.get(f"config{cfg_id}_{prec}", {}).get("k_forward_bytes_per_launch")
    except Exception:
        return None


def run_caller(cfg_id):
    """The SIP's caller on the config grid (one block, one GPU): assemble_poisson
    (periodic x / y, walls z), one factorisation, then pressure_correct outer
    iterations of 5 SIP sweeps each.
    Timed end to end per call (the call syncs once per outer iteration for the
    mass check); the SIP share from the library's CUDA-event profile."""
    import torch

    import paper_1303_4538_b200 as sip

    c = CONFIGS[cfg_id]
    g = tuple(c["g"])
    outer, sweeps = 4, 5
    s = sip.Solver(None, "f64", 0, lattice=(g, (1, 1, 1)))
    s.assemble_poisson((1.0, 1.0, 1.0), ("periodic", "periodic", "periodic", "periodic", "wall", "wall"))
    s.factor(0.92)
    fl = sip.Flow(s)
    (_, d, o) = s.blocks[0]
    x = (np.arange(d[0]) + 0.5) / g[0]
    z = (np.arange(d[2]) + 0.5) / g[2]
    for name, amp in zip("uvwp", (1.0, 0.0, 0.5, 0.0)):
        f = sip.field(*d)
        f[1:-1, 1:-1, 1:-1] = amp * np.sin(2 * np.pi * x)[None, None, :] * np.cos(np.pi * z)[:, None, None]
        fl.set(name, [f])
    ms = []
    for rep in range(3):  # rep 0 warms up
        s.set_profiling(True)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        try:
            fl.pressure_correct(0.01, 0.0, outer, sweeps)
        except sip.NonConvergenceError:
            pass  # threshold 0: the cap is the point
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        pr = s.profile()
        s.set_profiling(False)
        if rep:
            ms.append((wall * 1e3, pr["fwd_ms"] + pr["bwd_ms"] + pr["halo_ms"]))
    fl.close()
    s.close()
    wall_ms = statistics.median(m[0] for m in ms) / outer
    sip_ms = statistics.median(m[1] for m in ms) / outer
    cells = g[0] * g[1] * g[2]
    return {"workload": f"pressure_correct {g[0]}x{g[1]}x{g[2]} fp64, periodic x/y, walls z",
            "sweeps_per_outer": sweeps, "ms_per_outer": wall_ms, "sip_ms_per_outer": sip_ms,
            "caller_ms_per_outer": wall_ms - sip_ms,
            "sip_mlups": cells * sweeps / (sip_ms * 1e-3) / 1e6, "factorizations": 1}


def spawn(args) -> int:
    """--gpus N without a launcher: re-run this script under torchrun, one
    rank per GPU (fails loudly when fewer than N GPUs are visible)."""
    import socket

    import torch

    n = args.gpus
    have = torch.cuda.device_count()
    if have < n:
        print(f"bench.py: --gpus {n} but only {have} CUDA device(s) visible", file=sys.stderr)
        return 2
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def reference_line(args, world):
    cfg_id = args.config if args.config is not None else (1 if world == 1 else 3)
    c = CONFIGS[cfg_id]
    vals = []
    base = None
    t_all = time.perf_counter()
    for _ in range(args.steps):
        base = cpu_reference(cfg_id, seconds=max(2.0, 20.0 / max(1, args.steps)))
        vals.append(base["value"])
    v = statistics.median(vals)
    base["value"] = v
    return {"metric": "SIP inner-iteration MLUP/s", "value": v, "unit": "MLUP/s",
            "impl": "reference", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "higher_is_better": True, "scaling": "weak" if cfg_id != 4 else "strong",
            "dtype": c["prec"][0], "data": "synthetic (seeded generator, SURVEY.md 8(d))",
            "config": config_keys(cfg_id, world), "vs_baseline": None, "cpu_baseline": base,
            "e2e": {"value": v, "unit": "MLUP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "wall_s": time.perf_counter() - t_all}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=None)
    ap.add_argument("--precision", default="auto", choices=["auto", "f64", "f32"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-caller", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="N=1: skip the config 2/3/4 sub-objects")
    args = ap.parse_args()

    launched = "WORLD_SIZE" in os.environ
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.impl == "reference":
        # reference arm: CPU SIP on host cores, rank 0 only (others exit 0)
        if rank == 0:
            print(json.dumps(reference_line(args, max(world, args.gpus))), flush=True)
        return
    if not launched and args.gpus > 1:
        sys.exit(spawn(args))
    if launched and world != args.gpus:
        print(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}", file=sys.stderr)
        sys.exit(2)
    # NCCL's own init log names the communicator size (driver check of N ranks)
    os.environ.setdefault("NCCL_DEBUG", "INFO")
    dist = None
    if world > 1:
        import torch.distributed as dist_mod

        dist_mod.init_process_group("gloo", rank=rank, world_size=world)
        dist = dist_mod

    import torch

    import paper_1303_4538_b200 as sip

    sip.lib()  # fail loudly if the native library is missing
    torch.cuda.set_device(0 if world == 1 else int(os.environ.get("LOCAL_RANK", rank)))
    # a dedicated (non-default) stream: the library launches on it and the CUDA
    # events are recorded on it
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    cfg_id = args.config if args.config is not None else (1 if world == 1 else 3)
    c = CONFIGS[cfg_id]
    precs = c["prec"] if args.precision == "auto" else (args.precision,)
    res = {}
    for prec in precs:
        # e2e over 20 steps: the first step of a pipelined run cannot overlap its uploads
        # (pipeline fill, ~46 vs ~39 ms at config 1 fp64), inside the timed region
        res[prec] = measure(cfg_id, prec, rank, world, dist, stream, args.steps, args.warmup,
                            0 if args.no_e2e else 20)
    head = "f64" if "f64" in res else list(res)[0]
    r = res[head]
    # Eq. 1 efficiency: T_s from rank 0 alone on one GPU (the whole job for
    # strong scaling; one GPU's share x N for weak scaling)
    eff = None
    if world > 1:
        t1 = None
        if rank == 0:
            r1 = measure(cfg_id, head, 0, 1, None, stream, args.steps, 1)
            t1 = r1["ms"]
        obj = [t1]
        dist.broadcast_object_list(obj, src=0)
        t1 = obj[0]
        strong = cfg_id == 4
        t_s = t1 if strong else world * t1
        eff = {"eq": "perf.cpp Eq. 1: eps = T_s / (N * T_p(N))", "scaling": "strong" if strong else "weak",
               "t_s_ms": t_s, "t_p_ms": r["ms"], "n": world, "eps": t_s / (world * r["ms"]),
               "t1_source": "rank 0 alone, " + ("whole job" if strong else "one GPU's share") + ", same run"}
    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu:
            cpu = cpu_reference(cfg_id, seconds=12.0)
        caller = None
        if world == 1 and not args.no_caller and cfg_id == 1:
            caller = run_caller(cfg_id)
        extra = None
        if world == 1 and cfg_id == 1 and not args.no_extra and args.config is None:
            extra = {}
            for xc in (2, 3, 4):
                xp = CONFIGS[xc]["prec"][0]
                extra[f"config{xc}"] = summary(measure(xc, xp, 0, 1, None, stream, 2, 1), xc, xp)
        line = {
            "metric": "SIP inner-iteration MLUP/s", "value": r["value"], "unit": "MLUP/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": r["ms"], "higher_is_better": True,
            "scaling": "strong" if cfg_id == 4 and world > 1 else "weak",
            "vs_baseline": None, "dtype": head, "data": "synthetic (seeded generator, SURVEY.md 8(d))",
            "config": config_keys(cfg_id, world),
            "layout": {"bricks": r["geometry"], "parallelism": f"blocks over {world} GPU(s)"},
            "roofline": r["roofline"], "cpu_baseline": cpu, "e2e": r["e2e"],
            "gpu_launches": r["launches"], "clocks": r["clocks"],
            "achieved_hbm_gbs_step": r["step_gbs"], "achieved_frac_step": r["step_frac"],
            "k3_backward": r["k3"], "halo_ms_per_iter": r["halo_ms"],
            "kernel_ms_per_iter": r["kernel_ms_per_iter"],
            "timed_ms_per_iter": r["ms"] / c["iters"],
            "first_norms": r["first_norms"],
            "efficiency": eff,
            "caller": caller,
            "configs": extra,
        }
        for prec, rr in res.items():
            if prec == head:
                continue
            line[prec] = {"value": rr["value"], "ms_per_step": rr["ms"], "roofline": rr["roofline"],
                          "k3_backward": rr["k3"], "achieved_hbm_gbs_step": rr["step_gbs"],
                          "achieved_frac_step": rr["step_frac"], "e2e": rr["e2e"],
                          "gpu_launches": rr["launches"], "clocks": rr["clocks"]}
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
