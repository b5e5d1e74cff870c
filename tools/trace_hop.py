"""Cross-tile hop latency (globaltimer): trace tile W, then its east neighbour
T in a second identical run.  Per step s of T: W's publish of step s+15,
T's fetch of record s, T's loader announce of record s, T's prep(s) done."""
import ctypes, sys, os
import numpy as np
sys.path.insert(0, ".")
import paper_1303_4538_b200 as sip
g = (256, 256, 256)
prec = sys.argv[2] if len(sys.argv) > 2 else "f64"
def run(tile):
    os.environ["SIPB_TRACE_TILE"] = str(tile)
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
    tab = tr[:8 * nt.value].reshape(2, nt.value, 4).astype(np.int64)
    st = tr[8 * nt.value:].reshape(ns, 16).astype(np.int64)
    s.close()
    t0 = tab[0, :, 0].min()
    return tab, (st - t0) / 1e3, t0
W = int(sys.argv[1]) if len(sys.argv) > 1 else 17
T = W + 1
tabW, sW, _ = run(W)
tabT, sT, _ = run(T)
print("W", W, "start/end", (tabW[0, W, 0] - tabW[0, :, 0].min()) / 1e3, (tabW[0, W, 1] - tabW[0, :, 0].min()) / 1e3)
print("T", T, "start/end", (tabT[0, T, 0] - tabT[0, :, 0].min()) / 1e3, (tabT[0, T, 1] - tabT[0, :, 0].min()) / 1e3)
print("  s   Wpub(s+15)  Tfetch(s)  Tannounce(s)  Tprepdone(s)  Tissue(s)")
for s in (5, 10, 20, 40, 80, 120, 160, 200, 240, 270):
    print(f"{s:4d} {sW[s+15,12]:10.2f} {sT[s,9]:10.2f} {sT[s,10]:12.2f} {sT[s-1,3]:12.2f} {sT[s,8]:10.2f}")
