"""Device timeline of the split exchange (SIPB_XSPLIT=1): the span of one K3
sweep (its bricks' globaltimer start / end) and of the phase-1 copy kernel's
CTAs (first item start, last item end), on a block lattice with local copies
or, with SIPB_NCCL_SELF=1, NCCL packs.  Prints how much of the copy kernel's
active time falls inside K3's span.
usage: SIPB_XSPLIT=1 python tools/xsplit_timeline.py [f64|f32] [nxXnyXnz] [pxXpyXpz]"""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, ".")
os.environ.setdefault("SIPB_XSPLIT", "1")
import paper_1303_4538_b200 as sip  # noqa: E402

prec = sys.argv[1] if len(sys.argv) > 1 else "f64"
g = tuple(int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "256x256x256").split("x"))
pd = tuple(int(x) for x in (sys.argv[3] if len(sys.argv) > 3 else "2x2x2").split("x"))
s = sip.Solver(None, prec, 0, lattice=(g, pd))
s.generate(0, 1306)
s.factor(0.92)
s.load_phi([sip.field(*d) for (_, d, _) in s.blocks])
nt = ctypes.c_longlong()
L = sip.lib()
L.sip_debug_trace(s.handle, None, ctypes.byref(nt))
s.iterate(3)
buf = np.zeros(8 * nt.value + 5 * 64 * 6 + 2 * 256, dtype=np.uint64)
L.sip_debug_trace(s.handle, buf.ctypes.data_as(ctypes.POINTER(ctypes.c_ulonglong)), ctypes.byref(nt))
n = nt.value
k2 = buf[:4 * n].reshape(n, 4).astype(np.int64)
k3 = buf[4 * n:8 * n].reshape(n, 4).astype(np.int64)
xc = buf[8 * n + 5 * 64 * 6:].reshape(256, 2).astype(np.int64)
xc = xc[(xc[:, 0] > 0) & (xc[:, 1] > 0)]
t0 = k2[:, 0].min()
us = lambda v: (v - t0) / 1e3
k3s, k3e = us(k3[:, 0].min()), us(k3[:, 1].max())
cs, ce = us(xc[:, 0]), us(xc[:, 1])
inside = np.clip(np.minimum(ce, k3e) - np.maximum(cs, k3s), 0, None).sum() / max(1e-9, (ce - cs).sum())
print(f"{prec} {g} blocks {pd} (nccl_self={os.environ.get('SIPB_NCCL_SELF', '0')}): last sweep, us from its K2 start")
print(f"  K2 {us(k2[:, 0].min()):.1f} .. {us(k2[:, 1].max()):.1f}, K3 {k3s:.1f} .. {k3e:.1f}")
print(f"  phase-1 copy CTAs ({len(xc)}): first start {cs.min():.1f}, last end {ce.max():.1f}; "
      f"{100 * inside:.0f} % of their active time inside K3")
s.close()
