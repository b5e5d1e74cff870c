"""Per-brick end-time map of one K2 and one K3 sweep (single 256^3 block, brick trace
(library built with EXTRA=-DSIPB_STAGE_MARKS or plain; uses sip_debug_trace)): mean
gradient of the end time along i and j, i.e. the per-brick-hop cost of the wavefront.
usage: python tools/fill_map.py"""
import ctypes, sys
import numpy as np
sys.path.insert(0, ".")
import paper_1303_4538_b200 as sip
for prec in ("f64", "f32"):
    n = 256
    s = sip.Solver(None, prec, 0, lattice=((n, n, n), (1, 1, 1)))
    s.generate(0, 1304); s.factor(0.92); s.load_phi([sip.field(n, n, n)])
    nt = ctypes.c_longlong(); L = sip.lib()
    L.sip_debug_trace(s.handle, None, ctypes.byref(nt))
    s.iterate(3)
    buf = np.zeros(8 * nt.value + 5 * 64 * 6 + 2 * 256, dtype=np.uint64)
    L.sip_debug_trace(s.handle, buf.ctypes.data_as(ctypes.POINTER(ctypes.c_ulonglong)), ctypes.byref(nt))
    tr = buf[:8 * nt.value].reshape(2, nt.value, 4).astype(np.int64)
    BX, BY = 32, 8
    for kind, name in ((0, "K2"), (1, "K3")):
        t = tr[kind]; t0 = t[:, 0].min()
        en = ((t[:, 1] - t0) / 1e3).reshape(BY, BX)
        st = ((t[:, 0] - t0) / 1e3).reshape(BY, BX)
        dur = en - st
        # K2: wavefront from (0,0); K3 from (BX-1, BY-1)
        if kind == 1:
            en = en[::-1, ::-1]
        di = np.diff(en, axis=1); dj = np.diff(en, axis=0)
        print(f"{prec} {name}: span {en.max():.1f} us; end(0,0) {en[0,0]:.1f} end(last) {en[-1,-1]:.1f}; brick dur med {np.median(dur):.1f}")
        print("   mean d_end/d_i by row j:", " ".join(f"{x:.2f}" for x in di.mean(axis=1)))
        print("   mean d_end/d_j by col group:", " ".join(f"{x:.2f}" for x in dj.mean(axis=1)))
        print("   end row j=0 (every 4th):", " ".join(f"{x:.0f}" for x in en[0, ::4]))
        print("   end col i=0:", " ".join(f"{x:.0f}" for x in en[:, 0]))
        print("   end row j=7 (every 4th):", " ".join(f"{x:.0f}" for x in en[7, ::4]))
    s.close()
