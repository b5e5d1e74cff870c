"""Per-step pace of chosen tiles in one forward sweep (needs a -DSIPB_STEP_TRACE
build, e.g. make -C paper_1303_4538_b200/csrc exp NAME=trace EXTRA=-DSIPB_STEP_TRACE
and SIPB_LIB=exp/libsip_trace.so).  Prints, per tile, the global time of
steps 0, 16, 32, ... relative to the sweep start."""
import ctypes, os, sys
import numpy as np
sys.path.insert(0, ".")
import paper_1303_4538_b200 as sip
prec = sys.argv[1] if len(sys.argv) > 1 else "f64"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 256
TX = (n + 15) // 16
L = sip.lib()
ns = n + 30
for a in (0, 1, 2, 4, 8, 15):
    tile = a * TX + a
    os.environ["SIPB_TRACE_TILE"] = str(tile)
    s = sip.Solver(None, prec, 0, lattice=((n, n, n), (1, 1, 1)))
    s._nglobal = 1
    s.generate(0, 1304); s.factor(0.92); s.load_phi([sip.field(n, n, n)])
    nt = ctypes.c_longlong()
    L.sip_debug_trace(s.handle, None, ctypes.byref(nt))
    s.iterate(2)
    buf = np.zeros(8 * nt.value + 16 * ns, dtype=np.uint64)
    L.sip_debug_trace(s.handle, buf.ctypes.data_as(ctypes.POINTER(ctypes.c_ulonglong)), ctypes.byref(nt))
    tr = buf[:8 * nt.value].reshape(2, nt.value, 4).astype(np.int64)
    t0 = tr[1, :, 0].min()  # the forward sweep's table is the second half? use min over both
    t0 = min(tr[0, :, 0].min(), t0)
    st = buf[8 * nt.value:].reshape(ns, 16)[:, 0].astype(np.int64)
    fw0 = tr[0, :, 0].min()
    rel = (st - fw0) / 1e3
    marks = list(range(0, ns, 16)) + [ns - 1]
    print(f"tile ({a},{a}): " + " ".join(f"{rel[m]:.0f}" for m in marks))
    d = np.diff(st[32:ns - 32]) / 1e3
    print(f"   per-step pace median {np.median(d)*1e3:.0f} ns, mean {d.mean()*1e3:.0f} ns, p90 {np.percentile(d, 90)*1e3:.0f} ns")
    s.close()
