import sys, json, os
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np
import paper_1303_4538_b200 as sip
from oracle import oracle as O
import test_gpu_parity as T
gold = "tests/golden/ftt1"
name = "perx_2x2x1_r1"
f = json.load(open(os.path.join(gold, "cases.json")))["files"][name]
g, pd, mask = tuple(f["g"]), tuple(f["p"]), f["periodic_mask"]
tables = sip.ftt1_read(open(os.path.join(gold, name + ".ftt1"), "rb").read())
origins, dims, nbr = O.lattice(g, pd)
px, py, pz = pd
wrapped = []
for b in range(len(dims)):
    bx, by, bz = b % px, (b // px) % py, b // (px * py)
    bid = lambda x, y, z: (x % px) + px * ((y % py) + py * (z % pz))
    n = list(nbr[b])
    for axis in range(3):
        if (mask >> axis) & 1:
            lo = [bx, by, bz]; hi = [bx, by, bz]; lo[axis] -= 1; hi[axis] += 1
            n[2 * axis], n[2 * axis + 1] = bid(*lo), bid(*hi)
    wrapped.append(tuple(n))
print(wrapped)
s = sip.Solver(None, "f64", 0, lattice=(g, pd))
As = []
for lb, (bid_, d, o) in enumerate(s.blocks):
    A = T._periodic_system(O.generate(0, 1303 + 7 + bid_, d, g, o), d, o, g, mask)
    As.append(A); s.set_system(lb, sip.StencilSystem.from_dict(A))
s.set_halo_tables(tables); s.factor(0.92)
phis = [O.field(*d) for (_, d, _) in s.blocks]
s.load_phi(phis); s.iterate(6); s.store_phi(phis)
blocks = [(As[b], O.field(*dims[b])) for b in range(len(dims))]
no, _ = O.solve_multi(blocks, wrapped, 0.92, 6, "f64")
for b in range(len(dims)):
    a, r = phis[b], blocks[b][1]
    diff = np.argwhere(a != r)
    print(b, len(diff), "interior equal:", np.array_equal(a[1:-1,1:-1,1:-1], r[1:-1,1:-1,1:-1]), diff[:5].tolist())
    if len(diff): k,j,i = diff[0]; print("  gpu", a[k,j,i], "oracle", r[k,j,i])
