"""Wavefront drift along brick rows of one K2 and one K3 sweep (library built with
EXTRA=-DSIPB_STAGE_MARKS): per brick the time its stage kL/kStage completed
(early) and its end, along the row that starts the sweep (K2: j = 0, K3: j = BY-1)
and a middle row.  lag(early) = the wavefront skew a hop adds at the start;
lag(end) - lag(early) = the drift the hop accumulates over the brick.
usage: SIPB_LIB=exp/libsip_marks.so python tools/drift_map.py [f64|f32] [n]"""
import ctypes
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_1303_4538_b200 as sip  # noqa: E402

prec = sys.argv[1] if len(sys.argv) > 1 else "f64"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 256
s = sip.Solver(None, prec, 0, lattice=((n, n, n), (1, 1, 1)))
s.generate(0, 1304)
s.factor(0.92)
s.load_phi([sip.field(n, n, n)])
nt = ctypes.c_longlong()
L = sip.lib()
L.sip_debug_trace(s.handle, None, ctypes.byref(nt))
s.iterate(3)
buf = np.zeros(8 * nt.value + 5 * 64 * 6 + 2 * 256, dtype=np.uint64)
L.sip_debug_trace(s.handle, buf.ctypes.data_as(ctypes.POINTER(ctypes.c_ulonglong)), ctypes.byref(nt))
tr = buf[:8 * nt.value].reshape(2, nt.value, 4).astype(np.int64)
BX, BY = (n + 7) // 8, (n + 31) // 32
for kind, name in ((0, "K2"), (1, "K3")):
    t = tr[kind]
    t0 = t[:, 0].min()
    early = ((t[:, 3] - t0) / 1e3).reshape(BY, BX)
    end = ((t[:, 1] - t0) / 1e3).reshape(BY, BX)
    if kind == 1:
        early, end = early[::-1, ::-1], end[::-1, ::-1]
    for j in (0, BY // 2):
        le, ln = np.diff(early[j]), np.diff(end[j])
        print(f"{prec} {name} row {j}: early {early[j, 0]:.1f} -> {early[j, -1]:.1f} us, end {end[j, 0]:.1f} -> "
              f"{end[j, -1]:.1f} us; per hop: skew {le.mean():.2f} us, drift {np.mean(ln - le):.2f} us")
    print("   first 8 hops  skew:", " ".join(f"{x:.2f}" for x in np.diff(early[0])[:8]))
    print("   first 8 hops drift:", " ".join(f"{x:.2f}" for x in (np.diff(end[0]) - np.diff(early[0]))[:8]))
s.close()
