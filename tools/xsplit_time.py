"""Iteration time of multi-block contexts with the split exchange on / off
(SIPB_XSPLIT) and with the NCCL self-exchange (SIPB_NCCL_SELF): config 3
(8 x 128^3, fp64) and config 4 (128 x 128^3, fp32) on one GPU.

usage: python tools/xsplit_time.py [iters]
Prints per configuration: ms per iteration (wall clock over `iters`
iterations after a synchronize, device-bound) and the profiled K2 / K3 /
exposed-halo split."""
import os
import sys
import time

sys.path.insert(0, ".")

ITERS = int(sys.argv[1]) if len(sys.argv) > 1 else 40
CASES = [("config3", (256, 256, 256), (2, 2, 2), "f64"), ("config4", (1024, 512, 512), (8, 4, 4), "f32")]


def run(name, g, pd, prec, split, selfx):
    os.environ["SIPB_XSPLIT"] = "1" if split else "0"
    os.environ["SIPB_NCCL_SELF"] = "1" if selfx else "0"
    import paper_1303_4538_b200 as sip
    import torch

    s = sip.Solver(None, prec, 0, lattice=(g, pd))
    s.generate(0, 1306)
    s.factor(0.92)
    s.load_phi([sip.field(*d) for (_, d, _) in s.blocks])
    s.iterate(3)
    s.synchronize()
    t0 = time.perf_counter()
    s.iterate(ITERS)
    s.synchronize()
    wall = (time.perf_counter() - t0) * 1e3 / ITERS
    s.set_profiling(True)
    s.iterate(10)
    p = s.profile()
    s.close()
    torch.cuda.synchronize()
    print(f"{name} {prec} split={int(split)} nccl_self={int(selfx)}: {wall:.3f} ms/iter  "
          f"(K2 {p['fwd_ms'] / 10:.3f}, K3 {p['bwd_ms'] / 10:.3f}, exposed halo {p['halo_ms'] / 10:.3f})",
          flush=True)


for name, g, pd, prec in CASES:
    for selfx in ((False, True) if name == "config3" else (False,)):
        for split in (False, True):
            run(name, g, pd, prec, split, selfx)
