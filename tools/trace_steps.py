"""Per-step timing of one tile's forward sweep (SIPB_TRACE_TILE), config-1 sizes."""
import ctypes, sys, os
import numpy as np
sys.path.insert(0, ".")
import paper_1303_4538_b200 as sip
prec = sys.argv[1] if len(sys.argv) > 1 else "f64"
g = tuple(int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "256x256x256").split("x"))
s = sip.Solver(None, prec, 0, lattice=(g, (1, 1, 1)))
s._nglobal = 1
s.generate(0, 1304)
s.factor(0.92)
s.load_phi([sip.field(*g)])
nt = ctypes.c_longlong()
L = sip.lib()
L.sip_debug_trace(s.handle, None, ctypes.byref(nt))
s.iterate(2)
ns = g[2] + 30
tr = np.zeros(8 * nt.value + 4 * ns, dtype=np.uint64)
L.sip_debug_trace(s.handle, tr.ctypes.data_as(ctypes.POINTER(ctypes.c_ulonglong)), ctypes.byref(nt))
tab = tr[:8 * nt.value].reshape(2, nt.value, 4).astype(np.int64)
st = tr[8 * nt.value:].reshape(ns, 4).astype(np.int64)
tile = int(os.environ.get("SIPB_TRACE_TILE", "0"))
t0 = tab[0, :, 0].min()
print(f"{g} {prec} tile {tile}: start {(tab[0,tile,0]-t0)/1e3:.1f} us end {(tab[0,tile,1]-t0)/1e3:.1f} us; fwd span {(tab[0,:,1].max()-t0)/1e3:.1f} us")
a = (st[:, 0] - t0) / 1e3; b = (st[:, 1] - t0) / 1e3; c = (st[:, 2] - t0) / 1e3
step = np.diff(a)
print("step time us: median %.3f mean %.3f p90 %.3f max %.3f" % (np.median(step), step.mean(), np.percentile(step, 90), step.max()))
print("wait FW (b-a) median %.3f mean %.3f ; wait edge (c-b) median %.3f mean %.3f" % (np.median(b - a), (b - a).mean(), np.median(c - b), (c - b).mean()))
for t in list(range(0, 12)) + list(range(100, 106)) + list(range(ns - 4, ns)):
    print(f"  t={t:3d} enter {a[t]:8.2f} fw {b[t]-a[t]:6.3f} edge {c[t]-b[t]:6.3f} next {a[t+1]-c[t] if t+1<ns else 0:6.3f}")
