"""Isolated single-tile forward timeline in SM cycles (clock64): compute thread 0
[0] step top [1] after critical [3] slot wait done [4] prep computed [5] E arrived
[6] before barrier [7] after barrier; loader [8] slice s issued [10] record s
announced [11] loader saw E(x); fetcher [9] record s fetched."""
import ctypes, sys, os
import numpy as np
sys.path.insert(0, ".")
import paper_1303_4538_b200 as sip
prec = sys.argv[1] if len(sys.argv) > 1 else "f64"
g = tuple(int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "16x16x256").split("x"))
s = sip.Solver(None, prec, 0, lattice=(g, (1, 1, 1)))
s._nglobal = 1
s.generate(0, 1304); s.factor(0.92); s.load_phi([sip.field(*g)])
nt = ctypes.c_longlong(); L = sip.lib()
L.sip_debug_trace(s.handle, None, ctypes.byref(nt))
s.iterate(3)
ns = g[2] + 30
tr = np.zeros(8 * nt.value + 16 * ns, dtype=np.uint64)
L.sip_debug_trace(s.handle, tr.ctypes.data_as(ctypes.POINTER(ctypes.c_ulonglong)), ctypes.byref(nt))
st = tr[8 * nt.value:].reshape(ns, 16).astype(np.int64)
b0 = st[100, 0]
print("t    top  critEnd  slotWait(t+1) prepDone Earr barrierIn barrierOut | issue(t) announce(t) loaderSawE(t) | fetched(t)")
for t in range(100, 110):
    r = st[t] - b0
    print(f"{t} {r[0]:6d} {r[1]:6d} {r[3]:8d} {r[4]:8d} {r[5]:6d} {r[6]:7d} {r[7]:8d} | {r[8]:6d} fwdone {r[14]:6d} annDone {r[13]:6d} {r[10]:8d} {r[11]:8d} | {r[9]:8d}")
d = np.diff(st[20:-20, 0]); print("median step cycles", np.median(d))
