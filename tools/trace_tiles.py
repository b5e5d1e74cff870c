"""Per-tile start/end times of one forward and one backward sweep (config 1)."""
import ctypes, sys
import numpy as np
sys.path.insert(0, ".")
import paper_1303_4538_b200 as sip
prec = sys.argv[1] if len(sys.argv) > 1 else "f64"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 256
s = sip.Solver(None, prec, 0, lattice=((n, n, n), (1, 1, 1)))
s._nglobal = 1
s.generate(0, 1304)
s.factor(0.92)
s.load_phi([sip.field(n, n, n)])
nt = ctypes.c_longlong()
L = sip.lib()
L.sip_debug_trace(s.handle, None, ctypes.byref(nt))
s.iterate(3)
ns = n + 30
buf = np.zeros(8 * nt.value + 16 * ns, dtype=np.uint64)  # table + per-step record (see sip_debug_trace)
L.sip_debug_trace(s.handle, buf.ctypes.data_as(ctypes.POINTER(ctypes.c_ulonglong)), ctypes.byref(nt))
tr = buf[:8 * nt.value].reshape(2, nt.value, 4)
TX = (n + 15) // 16
for kind, name in ((0, "forward"), (1, "backward")):
    t = tr[kind].astype(np.int64)
    t0 = t[:, 0].min()
    st = (t[:, 0] - t0) / 1e3; en = (t[:, 1] - t0) / 1e3
    dur = en - st
    print(f"{name}: span {en.max():.1f} us, tile dur min/med/max {dur.min():.1f}/{np.median(dur):.1f}/{dur.max():.1f} us, "
          f"last start {st.max():.1f} us, distinct SMs {len(set(t[:,2].tolist()))}")
    # along the diagonal
    diag = [a * TX + a for a in range(TX)]
    print("  diag starts:", " ".join(f"{st[x]:.0f}" for x in diag))
    print("  diag ends:  ", " ".join(f"{en[x]:.0f}" for x in diag))
    row0 = [a for a in range(TX)]
    print("  row0 starts:", " ".join(f"{st[x]:.0f}" for x in row0))
