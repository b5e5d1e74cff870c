"""Cycle breakdown of one tile's forward steps (SIPB_TRACE_TILE; clock64):
compute thread 0: [0] step top [1] critical [2] - [3] prep wait done [4] prep compute
[5] E arrive [6] prep end [7] after barrier; loader [8] slice issue [11] E(x) seen;
fetcher [9] record fetched [10] record announced."""
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
tr = np.zeros(8 * nt.value + 16 * ns, dtype=np.uint64)
L.sip_debug_trace(s.handle, tr.ctypes.data_as(ctypes.POINTER(ctypes.c_ulonglong)), ctypes.byref(nt))
st = tr[8 * nt.value:].reshape(ns, 16).astype(np.int64)
tile = int(os.environ.get("SIPB_TRACE_TILE", "0"))
names = ["critical", "-", "prep-wait", "prep-compute", "E-arrive", "prep-tail", "barrier"]
rows = st[1:ns - 1]
print(f"{g} {prec} tile {tile}: cycles per step (median / mean) over {len(rows)} steps")
tot = np.diff(st[:, 0])
print("   step total     %7.0f %7.0f" % (np.median(tot), tot.mean()))
for i, n in enumerate(names):
    dlt = rows[:, i + 1] - rows[:, i]
    print("   %-14s %7.0f %7.0f" % (n, np.median(dlt), dlt.mean()))
# relative to the compute's prep-wait end of step x ([3] in the row of step x-1)
base = st[:-1, 3]   # prep(x+1) wait done is stored in row x
x = np.arange(1, ns)
iss = st[x, 8]; fet = st[x, 9]; ann = st[x, 10]; ew = st[x - 1, 11]
ready = base
sel = slice(20, ns - 20)
print("   slice issue -> prep ready   median %7.0f" % np.median((ready - iss)[sel]))
print("   record fetched -> ready     median %7.0f" % np.median((ready - fet)[sel]))
print("   record announced -> ready  median %7.0f" % np.median((ready - ann)[sel]))
print("   loader saw E(x-1) -> issue(x+SF-1) median %7.0f" % np.median((st[x[sel] + 2, 8] - ew[sel])))
b0 = st[100, 0]
print("   raw timeline (cycles rel. to step 100 top):  top  prepwait  Earr  bar | loaderSawE(x) issue(x) | fetched(x) announced(x)")
for t in range(100, 108):
    r = st[t] - b0
    print(f"   t={t}: {r[0]:7d} {r[3]:7d} {r[5]:7d} {r[7]:7d} | {r[11]:7d} {r[8]:7d} | {r[9]:8d} {r[10]:7d}")
