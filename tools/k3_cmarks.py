"""K3 compute-warp timeline of one brick (library built with
EXTRA="-DSIPB_STAGE_MARKS -DSIPB_K3_CMARKS", SIPB_LIB=exp/libsip_cmarks.so,
SIPB_TRACE_BRICK=b): per stage the hand-over arrival (chain done), when the
receiving warp was ready at the barrier, and when it was past its full wait.
usage: python tools/k3_cmarks.py [f64|f32] [nxXnyXnz]"""
import ctypes
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_1303_4538_b200 as sip  # noqa: E402

prec = sys.argv[1] if len(sys.argv) > 1 else "f64"
dims = [int(x) for x in sys.argv[2].split("x")] if len(sys.argv) > 2 else [8, 32, 256]
s = sip.Solver(None, prec, 0, lattice=(tuple(dims), (1, 1, 1)))
s.generate(0, 1304)
s.factor(0.92)
s.load_phi([sip.field(*dims)])
nt = ctypes.c_longlong()
L = sip.lib()
L.sip_debug_trace(s.handle, None, ctypes.byref(nt))
s.iterate(3)
buf = np.zeros(8 * nt.value + 5 * 64 * 6 + 2 * 256, dtype=np.uint64)
L.sip_debug_trace(s.handle, buf.ctypes.data_as(ctypes.POINTER(ctypes.c_ulonglong)), ctypes.byref(nt))
mk = buf[8 * nt.value:8 * nt.value + 5 * 64 * 6].reshape(5, 64, 6).astype(np.int64)[4]
arr, ready, full, cst, cen = mk[:, 3], mk[:, 0], mk[:, 5], mk[:, 1], mk[:, 2]
r = range(8, 60)
per = [arr[m + 1] - arr[m] for m in r]
late = [ready[m + 1] - arr[m] for m in r]       # > 0: receiver reached the barrier after the hand-over
run = [arr[m + 1] - max(arr[m], ready[m + 1]) for m in r]  # receiver: barrier release -> its own hand-over
pre = [ready[m + 1] - full[m + 1] for m in r]   # receiver: past full -> ready at the barrier (loads etc.)
med = lambda v: float(np.median(v))
print(f"{prec} {dims}: period {med(per):.0f} cyc; receiver ready - sender arrive {med(late):.0f} cyc "
      f"(late in {sum(x > 0 for x in late)}/{len(late)} stages); release -> next arrive {med(run):.0f} cyc; "
      f"past full -> ready {med(pre):.0f} cyc")
chain = [cen[m] - cst[m] for m in r]
wake = [cst[m + 1] - arr[m] for m in r]          # sender's arrive -> receiver's chain start (hand-over)
tail = [arr[m] - cen[m] for m in r]              # chain end -> hand-over stores + arrive
print(f"  chain {med(chain):.0f} cyc; hand-over: arrive -> next chain start {med(wake):.0f} cyc, "
      f"chain end -> arrive {med(tail):.0f} cyc")
print("  per-stage period:", " ".join(str(x) for x in per[:24]))
print("  late:            ", " ".join(str(x) for x in late[:24]))
s.close()
