"""Time of the pressure-correction caller (sip_pressure_correct) on one GPU.

One outer iteration = mass check (u, v, w ghosts + divergence + Q scatter) +
`sweeps` SIP iterations from p' = 0 + p' gather + velocity / pressure update.
The loop runs `outer` iterations against threshold 0 (NonConvergenceError at
the cap is expected) on a seeded smooth field; the SIP share comes from the
library's CUDA-event profile.  Usage: python tools/flow_bench.py [n] [px py pz]
"""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_1303_4538_b200 as sip  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
pd = tuple(int(x) for x in sys.argv[2:5]) if len(sys.argv) > 4 else (1, 1, 1)
outer, sweeps = 4, 5
for prec in ("f64", "f32"):
    s = sip.Solver(None, prec, 0, lattice=((n, n, n), pd))
    s.assemble_poisson((1.0, 1.0, 1.0), ("periodic", "periodic", "periodic", "periodic", "wall", "wall"))
    s.factor(0.92)
    fl = sip.Flow(s)
    rng = np.random.default_rng(1)
    for name in "uvwp":
        arrs = []
        for (_, d, o) in s.blocks:
            f = sip.field(*d)
            x = (np.arange(d[0]) + o[0] + 0.5) / n
            f[1:-1, 1:-1, 1:-1] = np.sin(2 * np.pi * x)[None, None, :] * rng.uniform(0.5, 1.0)
            arrs.append(f)
        fl.set(name, arrs)
    for rep in range(2):  # rep 0 warms up
        s.set_profiling(True)
        t0 = time.perf_counter()
        try:
            fl.pressure_correct(0.01, 0.0, outer, sweeps)
        except sip.NonConvergenceError:
            pass
        wall = time.perf_counter() - t0
        pr = s.profile()
        s.set_profiling(False)
    cells = n ** 3
    sip_ms = pr["fwd_ms"] + pr["bwd_ms"] + pr["halo_ms"]
    print(json.dumps({
        "workload": f"pressure_correct {n}^3 blocks {pd} {prec}", "outer": outer, "sweeps": sweeps,
        "ms_per_outer": round(wall * 1e3 / outer, 3),
        "sip_ms_per_outer": round(sip_ms / outer, 3),
        "caller_ms_per_outer": round(wall * 1e3 / outer - sip_ms / outer, 3),
        "sip_glups": round(cells * sweeps * outer / (sip_ms * 1e-3) / 1e9, 2),
    }))
    fl.close()
    s.close()
