"""Anatomy of one tile hop (tile A = $SIPB_TRACE_TILE -> tile A+1, 256^3, one forward sweep); needs
a -DSIPB_STEP_TRACE build (SIPB_LIB=exp/libsip_trace.so).  Tile 1's record s
carries tile 0's step s+15 output.  Prints medians of: A step -> A published,
published -> B fetched, fetched -> announced, announced -> B step s."""
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
A, B, pub, fet, ann = st[:, 0], st[:, 1], st[:, 2], st[:, 3], st[:, 4]
x = np.arange(40, ns - 40)
a = x + 15
def med(v): return f"{np.median(v):7.2f} (p90 {np.percentile(v, 90):6.2f})"
print(f"{prec} {n}^3: A pace {np.median(np.diff(A[40:-40]))*1e3:.0f} ns, B pace {np.median(np.diff(B[40:-40]))*1e3:.0f} ns")
print("  A step s+15 done -> A published   ", med(pub[a] - A[a]))
print("  A published      -> B fetched rec s", med(fet[x] - pub[a]))
print("  B fetched        -> B announced    ", med(ann[x] - fet[x]))
print("  B announced      -> B step s done  ", med(B[x] - ann[x]))
print("  total A step s+15 -> B step s      ", med(B[x] - A[a]))
print("startup (us): A step 0/15/16:", f"{A[0]:.2f} {A[15]:.2f} {A[16]:.2f}",
      "| A published 15/16:", f"{pub[15]:.2f} {pub[16]:.2f}",
      "| B fetched rec 0/1:", f"{fet[0]:.2f} {fet[1]:.2f}", "| B announced 0/1:", f"{ann[0]:.2f} {ann[1]:.2f}",
      "| B step 0/1/2:", f"{B[0]:.2f} {B[1]:.2f} {B[2]:.2f}")
for x in (20, 60, 120):
    print(f"  s={x}: A step s+15 {A[x+15]:.2f} pub {pub[x+15]:.2f} | B fetched {fet[x]:.2f} ann {ann[x]:.2f} step {B[x]:.2f}")
