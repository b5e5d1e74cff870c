"""Per-step timing of one tile's forward sweep (SIPB_TRACE_TILE): for step x,
trace[x] = {prep start, FW slice ready, edge record ready, phi ready}."""
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
a, b, c, e = [(st[:, i] - t0) / 1e3 for i in range(4)]
step = np.diff(a)
ok = st[:, 3] > 0
print("prep-to-prep us: median %.3f mean %.3f p90 %.3f" % (np.median(step), step.mean(), np.percentile(step, 90)))
print("wait FW median %.3f mean %.3f | wait edge median %.3f mean %.3f | wait phi median %.3f mean %.3f (active steps)" % (
    np.median(b - a), (b - a).mean(), np.median(c - b), (c - b).mean(), np.median((e - c)[ok]), (e - c)[ok].mean()))
for t in list(range(0, 6)) + list(range(100, 104)):
    print(f"  x={t:3d} start {a[t]:8.2f} fw {b[t]-a[t]:6.3f} edge {c[t]-b[t]:6.3f} phi {(e[t]-c[t]) if ok[t] else 0:6.3f} rest {a[t+1]-max(c[t], e[t]):6.3f}")
