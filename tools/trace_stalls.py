"""Poll stalls per tile (events, stalled time summed over the tile's edge
threads) of one forward and one backward sweep; needs a -DSIPB_STEP_TRACE
build (SIPB_LIB=exp/libsip_trace.so)."""
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
tr = buf[:8 * nt.value].reshape(2, nt.value, 4)
TX = (n + 15) // 16
for kind, name in ((0, "forward"), (1, "backward")):
    v = tr[kind, :, 3]
    ev = (v >> np.uint64(40)).astype(np.int64)
    tns = (v & np.uint64((1 << 40) - 1)).astype(np.int64)
    dur = (tr[kind, :, 1].astype(np.int64) - tr[kind, :, 0].astype(np.int64)) / 1e3
    print(f"{name}: stall events per tile median {np.median(ev):.0f} max {ev.max()}, "
          f"stalled us per stalled thread-event median {np.median(tns[ev>0]/ev[ev>0])/1e3:.2f}")
    for a in (0, 1, 4, 8, 15):
        t = a * TX + a
        print(f"  tile ({a},{a}): events {ev[t]}, stalled {tns[t]/1e3:.1f} us (sum over threads), tile dur {dur[t]:.1f} us")
