"""Per-step wall time of the e2e call patterns at config 1 (256^3): sequential
(sip_set_source + sip_solve), one async solve pending, two in flight; for
`iters` sweeps per step (1: the transfers dominate).
usage: python tools/e2e_pipe.py [f64|f32] [iters] [steps]"""
import ctypes
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1303_4538_b200 as sip  # noqa: E402

prec = sys.argv[1] if len(sys.argv) > 1 else "f64"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 1
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 10
n = 256
s = sip.Solver(None, prec, 0, lattice=((n, n, n), (1, 1, 1)))
s.generate(0, 1304)
s.factor(0.92)
L = sip.lib()
dp = ctypes.POINTER(ctypes.c_double)
phi_t = torch.zeros((n + 2,) * 3, dtype=torch.float64).pin_memory()
q_t = torch.zeros((n + 2,) * 3, dtype=torch.float64).pin_memory()
q_t[1:-1, 1:-1, 1:-1] = 1.0
arr = (dp * 1)(phi_t.numpy().ctypes.data_as(dp))
qp = q_t.numpy().ctypes.data_as(dp)
nrm = [np.zeros(iters), np.zeros(iters)]
used = ctypes.c_int()


def seq(k):
    for _ in range(k):
        L.sip_set_source(s.handle, 0, qp)
        assert L.sip_solve(s.handle, arr, iters, ctypes.c_double(0.0), nrm[0].ctypes.data_as(dp),
                           ctypes.byref(used)) == 0


def one_pending(k):
    L.sip_set_source_async(s.handle, 0, qp)
    for r in range(k):
        assert L.sip_solve_async(s.handle, arr, iters, nrm[0].ctypes.data_as(dp)) == 0
        if r + 1 < k:
            L.sip_set_source_async(s.handle, 0, qp)
        L.sip_synchronize(s.handle)


STEP_T = []


def two(k):
    def enq(r):
        L.sip_set_source_async(s.handle, 0, qp)
        assert L.sip_solve_async(s.handle, arr, iters, nrm[r % 2].ctypes.data_as(dp)) == 0
    enq(0)
    t = time.perf_counter()
    for r in range(k):
        if r + 1 < k:
            enq(r + 1)
        L.sip_wait_async(s.handle)
        t2 = time.perf_counter()
        STEP_T.append((t2 - t) * 1e3)
        t = t2


def one_noq(k):
    for r in range(k):
        assert L.sip_solve_async(s.handle, arr, iters, nrm[0].ctypes.data_as(dp)) == 0
        L.sip_synchronize(s.handle)


def two_noq(k):
    assert L.sip_solve_async(s.handle, arr, iters, nrm[0].ctypes.data_as(dp)) == 0
    for r in range(k):
        if r + 1 < k:
            assert L.sip_solve_async(s.handle, arr, iters, nrm[(r + 1) % 2].ctypes.data_as(dp)) == 0
        L.sip_wait_async(s.handle)


for name, f in (("sequential", seq), ("one pending", one_pending), ("two in flight", two),
                ("one, no Q", one_noq), ("two, no Q", two_noq)):
    f(2)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    f(steps)
    torch.cuda.synchronize()
    print(f"{prec} iters={iters}: {name:14s} {(time.perf_counter() - t0) / steps * 1e3:7.2f} ms/step")
    if name == "two in flight":
        print("   per step:", " ".join(f"{x:.1f}" for x in STEP_T[-steps:]))
s.close()
