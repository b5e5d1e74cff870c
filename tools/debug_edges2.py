import ctypes, sys
import numpy as np
sys.path.insert(0, ".")
import paper_1303_4538_b200 as sip
from oracle import oracle as O
dp = ctypes.POINTER(ctypes.c_double)
dims = (32, 17, 19)
A = O.generate(0, 1303, dims)
F = O.factor(A, 0.92)
s = sip.Solver(dims, "f64")
s.set_system(0, sip.StencilSystem.from_dict(A))
s.factor(0.92)
s.load_phi([O.field(*dims)])
s.iterate(1)
pg = O.field(*dims); s.store_phi([pg])
po = O.field(*dims); O.sweep(A, F, po)
R = O.forward(A, F, O.field(*dims))
# consumer column: tile (0,1) cell (15,0) -> 1-based i=16, j=17; E neighbour i=17
for k in range(18, 10, -1):
    kk = k + 1
    dE_or = po[kk, 17, 17]
    dT_or = po[kk + 1, 17, 16] if k < 18 else 0.0
    d_gpu = pg[kk, 17, 16]
    r = R[kk, 17, 16]; ue = F["UE"][kk, 17, 16]; ut = F["UT"][kk, 17, 16]; un = F["UN"][kk, 17, 16]
    # solve for the dE the GPU must have used (assuming dN = 0 and its own dT)
    dT_gpu = pg[kk + 1, 17, 16] if k < 18 else 0.0
    dE_used = ((r - un * 0.0) - ut * dT_gpu - d_gpu) / ue if ue else float('nan')
    print(k, "dE oracle", dE_or, "dE used", dE_used, "d_gpu", d_gpu, "d_or", po[kk,17,16])
