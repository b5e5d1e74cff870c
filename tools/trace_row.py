"""Hop latency along one row of tiles (tiles 0..15 = (0,0)..(0,15) at 256^3)
in one forward sweep; needs a -DSIPB_STEP_TRACE build (SIPB_LIB=exp/libsip_trace.so).
Tile b+1 step s consumes tile b's step s+15 (geometric lag 16 steps): print the
time from tile b's step s+15 to tile b+1's step s."""
import ctypes, sys
import numpy as np
sys.path.insert(0, ".")
import paper_1303_4538_b200 as sip
prec = sys.argv[1] if len(sys.argv) > 1 else "f64"
n = 256
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
tr = buf[:8 * nt.value].reshape(2, nt.value, 4).astype(np.int64)
t0 = tr[0, :, 0].min()
st = (buf[8 * nt.value:].reshape(ns, 16).astype(np.int64) - t0) / 1e3  # [step][tile] us
print("tile step-0 times:", " ".join(f"{st[0, b]:.1f}" for b in range(16)))
print("tile last-step times:", " ".join(f"{st[ns - 1, b]:.0f}" for b in range(16)))
for b in (0, 1, 4, 8, 14):
    lagt = [st[x, b + 1] - st[x + 15, b] for x in range(0, ns - 15)]
    pace = np.diff(st[:, b + 1])
    print(f"hop {b}->{b+1}: (B step s) - (A step s+15): median {np.median(lagt):.2f} us, p10 {np.percentile(lagt,10):.2f}, p90 {np.percentile(lagt,90):.2f};"
          f" B pace median {np.median(pace)*1e3:.0f} ns mean {pace.mean()*1e3:.0f}")
