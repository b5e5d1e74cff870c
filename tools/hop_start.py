"""First stages of a K3 hop (library built with EXTRA=-DSIPB_STAGE_MARKS;
SIPB_TRACE_BRICK = the downstream brick, SIPB_TRACE_UP = its upstream offset):
per stage the upstream's cdone / publish and the downstream's poll start, value
seen, past full and cdone (us from the first mark).
usage: SIPB_LIB=exp/libsip_marks.so SIPB_TRACE_BRICK=b SIPB_TRACE_UP=1 python tools/hop_start.py [f64|f32] [n] [stages]"""
import ctypes
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_1303_4538_b200 as sip  # noqa: E402

prec = sys.argv[1] if len(sys.argv) > 1 else "f64"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 256
ns = int(sys.argv[3]) if len(sys.argv) > 3 else 16
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
tr = buf[:8 * nt.value].reshape(2, nt.value, 4).astype(np.int64)[1]
mk = buf[8 * nt.value:8 * nt.value + 5 * 64 * 6].reshape(5, 64, 6).astype(np.int64)
up, dn = mk[3], mk[4]
t0 = tr[:, 0].min()
f = lambda v: (v - t0) / 1e3 if v > 0 else float("nan")
print(f"{prec} {n}^3  K3 launch-relative times (us); cols: up cdone, up published | dn poll, dn seen, dn full, dn cdone")
for m in range(ns):
    print(f"  m={m:3d}  {f(up[m, 3]):7.2f} {f(up[m, 4]):7.2f} | {f(dn[m, 0]):7.2f} {f(dn[m, 1]):7.2f} "
          f"{f(dn[m, 2]):7.2f} {f(dn[m, 3]):7.2f}")
s.close()
