"""Compare R after one forward sweep (K2) with the oracle, per cell."""
import ctypes
import sys
import numpy as np
sys.path.insert(0, ".")
import paper_1303_4538_b200 as sip
from oracle import oracle as O

dp = ctypes.POINTER(ctypes.c_double)
cases = [tuple(int(x) for x in c.split("x")) for c in sys.argv[1:]] or [(17, 17, 3)]
for dims in cases:
    A = O.generate(0, 1303, dims)
    F = O.factor(A, 0.92)
    s = sip.Solver(dims, "f64")
    s.set_system(0, sip.StencilSystem.from_dict(A))
    s.factor(0.92)
    # factors identical?
    for w, n in [(10, "LB"), (11, "LW"), (12, "LS"), (13, "LP"), (14, "UN"), (15, "UE"), (16, "UT")]:
        out = O.field(*dims)
        sip.lib().sip_debug_field(s.handle, 0, w, out.ctypes.data_as(dp))
        dd = np.argwhere(out[1:-1, 1:-1, 1:-1] != F[n][1:-1, 1:-1, 1:-1])
        if len(dd):
            print(dims, "factor", n, "ndiff", len(dd), "first (k,j,i)", dd[0])
    phi = O.field(*dims)
    s.load_phi([phi])
    sip.lib().sip_debug_forward(s.handle)
    Rg = O.field(*dims)
    sip.lib().sip_debug_field(s.handle, 0, 1, Rg.ctypes.data_as(dp))
    Ro = O.forward(A, F, phi)
    dd = np.argwhere(Rg[1:-1, 1:-1, 1:-1] != Ro[1:-1, 1:-1, 1:-1])
    msg = f"{dims} forward R ndiff={len(dd)}"
    if len(dd):
        k, j, i = sorted(tuple(x) for x in dd)[0]
        msg += f" first lexicographic (i,j,k)=({i},{j},{k}) tile=({i//16},{j//16}) ti,tj=({i%16},{j%16})"
    print(msg, flush=True)
    # full iteration
    s2 = O.field(*dims)
    s.load_phi([s2])
    s.iterate(1)
    pg = O.field(*dims)
    s.store_phi([pg])
    po = O.field(*dims)
    O.sweep(A, F, po)
    dd = np.argwhere(pg[1:-1, 1:-1, 1:-1] != po[1:-1, 1:-1, 1:-1])
    msg = f"{dims} iteration phi ndiff={len(dd)}"
    if len(dd):
        k, j, i = sorted((tuple(x) for x in dd), reverse=True)[0]
        msg += f" first-in-backward (i,j,k)=({i},{j},{k}) tile=({i//16},{j//16}) ti,tj=({i%16},{j%16})"
    print(msg, flush=True)
    s.close()
