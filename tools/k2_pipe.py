"""K2 pipeline timing of one brick (library built with -DSIPB_STAGE_MARKS):
per stage, cycles between TMA issue, residual past full, residual / mailbox
ready, recurrence past ready, rdone.  usage: SIPB_LIB=... SIPB_TRACE_BRICK=b
python tools/k2_pipe.py [f64|f32] [n | nxXnyXnz]"""
import ctypes
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_1303_4538_b200 as sip  # noqa: E402

prec = sys.argv[1] if len(sys.argv) > 1 else "f64"
dims = [int(x) for x in sys.argv[2].split("x")] if len(sys.argv) > 2 else [256]
nx, ny, nz = dims if len(dims) == 3 else dims * 3
s = sip.Solver(None, prec, 0, lattice=((nx, ny, nz), (1, 1, 1)))
s.generate(0, 1304)
s.factor(0.92)
s.load_phi([sip.field(nx, ny, nz)])
nt = ctypes.c_longlong()
L = sip.lib()
L.sip_debug_trace(s.handle, None, ctypes.byref(nt))
s.iterate(3)
buf = np.zeros(8 * nt.value + 5 * 64 * 6 + 2 * 256, dtype=np.uint64)
L.sip_debug_trace(s.handle, buf.ctypes.data_as(ctypes.POINTER(ctypes.c_ulonglong)), ctypes.byref(nt))
mk = buf[8 * nt.value:8 * nt.value + 5 * 64 * 6].reshape(5, 64, 6).astype(np.int64)[2]
r = range(8, 60)
med = lambda v: float(np.median(v))
print(f"{prec} {nx}x{ny}x{nz} brick: stage period (rdone) {med(np.diff(mk[8:60, 5])):.0f} cycles")
names = ["TMA issued", "residual past full", "residual ready", "mailbox ready", "recurrence past ready", "rdone"]
for a, b in [(0, 1), (1, 2), (2, 4), (3, 4), (4, 5)]:
    print(f"  {names[a]:22s} -> {names[b]:22s} {med([mk[m, b] - mk[m, a] for m in r]):8.0f}")
for d in range(1, 5):
    print(f"  rdone(n-{d}) -> TMA issued(n)       {med([mk[m, 0] - mk[m - d, 5] for m in r]):8.0f}")
print(f"  TMA issued(n) -> rdone(n)             {med([mk[m, 5] - mk[m, 0] for m in r]):8.0f}")
s.close()
