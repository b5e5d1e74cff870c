"""Cross-tile hop latency: run the forward sweep tracing tile W, then tile T = W's
east neighbour (globaltimer stamps).  For step s of T: W published progress
s+16 at P_W[s+15]; T's fetcher saw it at F_T[s]; T's prep of step s ended at C_T[s]."""
import ctypes, sys, os, subprocess
import numpy as np
sys.path.insert(0, ".")
import paper_1303_4538_b200 as sip
g = (256, 256, 256)
def run(tile):
    os.environ["SIPB_TRACE_TILE"] = str(tile)
    s = sip.Solver(None, "f64", 0, lattice=(g, (1, 1, 1)))
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
    return tab, st
W = int(sys.argv[1]) if len(sys.argv) > 1 else 17   # tile (1,1)
T = W + 1                                            # tile (2,1)
tabW, stW = run(W)
tabT, stT = run(T)
# align each run to its own kernel start (min tile start); runs differ, so compare
# within-run quantities only, and W/T via the same reference
t0W = tabW[0, :, 0].min(); t0T = tabT[0, :, 0].min()
print("W start/end (us):", (tabW[0, W, 0] - t0W) / 1e3, (tabW[0, W, 1] - t0W) / 1e3)
print("T start/end (us):", (tabT[0, T, 0] - t0T) / 1e3, (tabT[0, T, 1] - t0T) / 1e3)
ns = stT.shape[0]
pubW = (stW[:, 12] - t0W) / 1e3   # W published progress s+1 at pubW[s]
fetT = (stT[:, 13] - t0T) / 1e3   # T's fetcher allowed record s
prepT = (stT[:, 3] - t0T) / 1e3   # T: prep(s+1) wait done (row s)
stepT = (stT[:, 0] - t0T) / 1e3
for s in (20, 50, 100, 150, 200, 250):
    print(f" s={s}: W pub(s+16) {pubW[s+15]:8.2f}  T fetch-allowed(s) {fetT[s]:8.2f}  T step(s) top {stepT[s]:8.2f}  T step period {stepT[s+1]-stepT[s]:.3f}")
print("T step period median (us):", np.median(np.diff(stepT[20:-20])))
print("W publish period median (us):", np.median(np.diff(pubW[20:-40])))
