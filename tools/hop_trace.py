"""Hand-off timing between a brick and its E neighbour (SIPB_TRACE_UP=1) or N
neighbour (SIPB_TRACE_UP=BX) in one backward sweep
(library built with EXTRA=-DSIPB_STAGE_MARKS; SIPB_TRACE_BRICK = the W brick).
usage: SIPB_LIB=exp/libsip_marks.so SIPB_TRACE_BRICK=b python tools/hop_trace.py [f64|f32] [n]"""
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
mk = buf[8 * nt.value:8 * nt.value + 5 * 64 * 6].reshape(5, 64, 6).astype(np.int64)
up, dn = mk[3], mk[4]
t0 = min(x for x in np.concatenate([up[:, :5].ravel(), dn[:, :5].ravel()]) if x > 0)
up = np.where(up > 0, up - t0, 0) / 1e3
dn = np.where(dn > 0, dn - t0, 0) / 1e3
r = range(8, 56)
med = lambda v: float(np.median(v))
print(f"{prec} {n}^3 brick {sys.argv[0]} stage period down {med(np.diff(dn[8:56, 3])):.3f} us, up {med(np.diff(up[8:56, 3])):.3f} us")
print("  up:   cdone -> published          %.3f us" % med([up[m, 4] - up[m, 3] for m in r]))
print("  down: poll start -> seen         %.3f us" % med([dn[m, 1] - dn[m, 0] for m in r]))
print("  down: seen -> compute past full  %.3f us" % med([dn[m, 2] - dn[m, 1] for m in r]))
print("  down: past full -> cdone         %.3f us" % med([dn[m, 3] - dn[m, 2] for m in r]))
for d in range(0, 7):
    print(f"  seen_down(m) - published_up(m+{d}) %.3f us" % med([dn[m, 1] - up[m + d, 4] for m in r]))
print("  cdone_down(m) - cdone_up(m)        %.3f us" % med([dn[m, 3] - up[m, 3] for m in r]))
s.close()
