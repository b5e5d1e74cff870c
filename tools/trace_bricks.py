"""Per-brick start/end times of one forward (K2) and one backward (K3) sweep.

usage: python tools/trace_bricks.py [f64|f32] [n | nxXnyXnz]   (single block, kind-0 system)
Prints the sweep span, brick duration stats, and the start / end times along
the first brick row (i direction) and column (j direction)."""
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
tr = buf[:8 * nt.value].reshape(2, nt.value, 4)
marks2 = buf[8 * nt.value:8 * nt.value + 5 * 64 * 6].reshape(5, 64, 6).astype(np.int64)
g = s.geometry()
BX = (nx + g["brick_i"] - 1) // g["brick_i"]
BY = (ny + g["brick_j"] - 1) // g["brick_j"]
slices = g["slices"] // nt.value
for kind, name in ((0, "forward"), (1, "backward")):
    t = tr[kind].astype(np.int64)
    t0 = t[:, 0].min()
    st = (t[:, 0] - t0) / 1e3
    en = (t[:, 1] - t0) / 1e3
    dur = en - st
    print(f"{name}: span {en.max():.1f} us, brick dur min/med/max {dur.min():.1f}/{np.median(dur):.1f}/"
          f"{dur.max():.1f} us ({1e3 * np.median(dur) / slices:.1f} ns/slice), last start {st.max():.1f} us, "
          f"SMs {len(set(t[:, 2].tolist()))}")
    row = list(range(BX))
    col = [BX * j for j in range(BY)]
    print("  row0 start:", " ".join(f"{st[x]:.0f}" for x in row))
    print("  row0 end:  ", " ".join(f"{en[x]:.0f}" for x in row))
    print("  col0 start:", " ".join(f"{st[x]:.0f}" for x in col))
    print("  col0 end:  ", " ".join(f"{en[x]:.0f}" for x in col))
    s4 = (t[:, 3] - t0) / 1e3  # end of the brick's stage 4 (first interior stage)
    print("  row0 stage4:", " ".join(f"{s4[x]:.0f}" for x in row))
    print("  col0 stage4:", " ".join(f"{s4[x]:.0f}" for x in col))
    last = BX * BY - 1
    print(f"  last brick start {st[last]:.0f} end {en[last]:.0f}")
for kk, marks in enumerate(marks2):
    if not marks[:, 0].any():
        continue
    nz = [i for i in range(6) if marks[8, i] != 0]
    if len(nz) < 2:
        continue
    marks = marks[:, nz]
    # per-stage marks of brick SIPB_TRACE_BRICK (cycles): validate, mbar wait, phase A, B, C
    d = np.diff(marks, axis=1)
    step = np.diff(marks[:, 0])
    print("%s stage marks (cycles, stages 8..63 median): %s  stage %.0f  (mean %s)" % (
        ("K2B", "K3C", "K2A", "P", "M")[kk], " ".join("%.0f" % x for x in np.median(d[8:], axis=0)), np.median(step[8:]),
        " ".join("%.0f" % x for x in np.mean(d[8:], axis=0))))
s.close()
