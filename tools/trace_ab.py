"""Tile hop A -> A+1 (A = $SIPB_TRACE_TILE) in one forward sweep at n^3: time
from A's step s+15 to B's step s (B's step s consumes A's step s+15 output;
ideal difference = one hyperplane step).  Needs a -DSIPB_STEP_TRACE build."""
import ctypes, sys
import numpy as np
sys.path.insert(0, ".")
import paper_1303_4538_b200 as sip
prec = sys.argv[1] if len(sys.argv) > 1 else "f64"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 256
ns = n + 30
s = sip.Solver(None, prec, 0, lattice=((n, n, n), (1, 1, 1)))
s._nglobal = 1
s.generate(0, 1304); s.factor(0.92); s.load_phi([sip.field(n, n, n)])
L = sip.lib()
nt = ctypes.c_longlong()
L.sip_debug_trace(s.handle, None, ctypes.byref(nt))
s.iterate(2)
buf = np.zeros(8 * nt.value + 16 * ns, dtype=np.uint64)
L.sip_debug_trace(s.handle, buf.ctypes.data_as(ctypes.POINTER(ctypes.c_ulonglong)), ctypes.byref(nt))
tr = buf[:8 * nt.value].reshape(2, nt.value, 4).astype(np.int64)
t0 = tr[0, :, 0].min()
st = (buf[8 * nt.value:].reshape(ns, 16).astype(np.int64) - t0) / 1e3
A, B = st[:, 0], st[:, 1]
x = np.arange(40, ns - 40)
dA, dB = np.diff(A[40:-40]), np.diff(B[40:-40])
print(f"{prec} {n}^3 tiles {tr[0,:,0].size}: A pace median {np.median(dA)*1e3:.0f} mean {dA.mean()*1e3:.0f} ns; "
      f"B pace median {np.median(dB)*1e3:.0f} mean {dB.mean()*1e3:.0f} ns")
v = B[x] - A[x + 15]
print(f"  A step s+15 -> B step s: median {np.median(v):.2f} us (p10 {np.percentile(v,10):.2f}, p90 {np.percentile(v,90):.2f})")
print(f"  A step 0 {A[0]:.2f}, A step 15 {A[15]:.2f}, B step 0 {B[0]:.2f}; A end {A[-1]:.1f}, B end {B[-1]:.1f}")
for nm, dd in (("A", dA), ("B", dB)):
    q = np.percentile(dd, [10, 50, 75, 90, 99]) * 1e3
    print(f"  {nm} step ns p10/50/75/90/99: {' '.join(f'{v:.0f}' for v in q)}")
# who waits: crit thread 0 reaches the end of step t-1 (slot 0 at t-1) vs the residual
# group publishing r(t) (slot 6 at t); positive = the critical group waits for the residual
R6 = st[:, 6]
if R6.max() > 0:
    w = R6[41:-40] - A[40:-41]
    print(f"  residual r(t) after crit end of t-1: median {np.median(w)*1e3:.0f} ns, "
          f"p90 {np.percentile(w,90)*1e3:.0f} ns, share of steps where crit waits {np.mean(w>0)*100:.0f}%")
S7 = st[:, 7]
if S7.max() > 0:
    inner = A[40:-40] - S7[40:-40]          # thread 0 inside step t (incl. its own W/S polls)
    wait = S7[41:-40] - A[40:-41]           # barrier wait after step t-1 (slowest thread / warp)
    print(f"  thread 0 in-step: median {np.median(inner)*1e3:.0f} ns p90 {np.percentile(inner,90)*1e3:.0f}; "
          f"barrier wait: median {np.median(wait)*1e3:.0f} ns p90 {np.percentile(wait,90)*1e3:.0f}")
