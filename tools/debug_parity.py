"""Locate the first cells where the GPU SIP path differs from the oracle."""
import sys
import numpy as np
sys.path.insert(0, ".")
import paper_1303_4538_b200 as sip
from oracle import oracle as O

cases = [tuple(int(x) for x in c.split("x")) for c in sys.argv[1:]] or [(21, 21, 19)]
for dims in cases:
    A = O.generate(0, 1303, dims)
    for alpha in (0.92, 0.0):
        s = sip.Solver(dims, "f64")
        s.set_system(0, sip.StencilSystem.from_dict(A))
        s.factor(alpha)
        pg = O.field(*dims)
        ng = s.solve([pg], 1)
        s.close()
        po = O.field(*dims)
        no = O.solve(A, po, alpha, 1, "f64")
        diff = np.argwhere(pg != po)
        msg = f"{dims} alpha={alpha} ndiff={len(diff)}"
        if len(diff):
            # cells sorted by reverse lexicographic (backward order): first wrong in backward order
            order = sorted([tuple(x) for x in diff], reverse=True)
            k, j, i = order[0]
            msg += f" first-in-backward (i,j,k)=({i},{j},{k}) tile=({(i-1)//16},{(j-1)//16}) maxdiff={np.abs(pg-po).max():.3e}"
        print(msg, flush=True)
