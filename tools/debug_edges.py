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
n = ctypes.c_longlong()
sip.lib().sip_debug_edges(s.handle, 0, None, ctypes.byref(n))
eW = np.zeros(n.value); sip.lib().sip_debug_edges(s.handle, 0, eW.ctypes.data_as(dp), ctypes.byref(n))
nz = dims[2]
# tiles: 0=(0,0) 1=(1,0) 2=(0,1) 3=(1,1); edge offset = tile * nz * 16
t = 3
for k in range(nz):
    v = eW[t * nz * 16 + k * 16 + 0]
    ref = po[k + 1, 17, 17]  # tile (1,1) cell (0,0) -> i=17, j=17 (1-based)
    gpu = pg[k + 1, 17, 17]
    print(k, v, ref, gpu, "OK" if v == ref else "DIFF")
# the consumer cell (15,0) of tile (0,1) -> i=16, j=17
print("consumer col diffs:", [(k, pg[k+1,17,16]-po[k+1,17,16]) for k in range(nz)][:5])
