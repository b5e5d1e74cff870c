"""Regenerate the committed golden fixtures under tests/golden/.

TEST INFRASTRUCTURE.  Run in the build container (needs /root/reference):

    python oracle/make_golden.py

1. ref_tables.json -- the reference's own block decomposition and face
   transfer tables (bsfv::decompose / with_ranks / build_transfer_tables,
   proj/src/grid.cpp, proj/src/transfers.cpp, proj/src/tables.cpp), produced
   by oracle/_ref/ref_tables_dump, which is compiled in place from the
   reference sources (oracle/Makefile target `ref`).  These pin the halo plan
   of the B200 library (sip_plan_halo) to the reference's behaviour.
3. perf_golden.txt -- the reference's own perf module (proj/src/perf.cpp,
   compiled in place into oracle/_ref/ref_perf_dump) over the scenarios of
   tests/golden/perf_scenarios.txt (Eq. 1, Eq. 2, threshold points,
   iso-efficiency, shortest round-trip formatting, error messages); pins
   include/bsfv_perf.hpp byte for byte.
2. sip_golden.npz -- oracle SIP outputs (norm histories, phi checksums) of
   small seeded systems.  The reference has no SIP code to run, so these are
   regression pins of the restatement (checked against the SPEC known-answer
   properties in tests/test_oracle.py), not reference outputs.
"""
from __future__ import annotations

import json
import os
import subprocess
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)
GOLD = os.path.join(ROOT, "tests", "golden")

TABLE_CASES = [
    # (grid, blocks, ranks)  ranks 0 = one block per rank
    ((8, 8, 8), (2, 1, 1), 0),
    ((8, 6, 4), (2, 2, 1), 0),
    ((8, 6, 4), (2, 2, 1), 2),
    ((5, 4, 4), (2, 1, 1), 0),     # remainder to the last block
    ((9, 7, 5), (3, 2, 2), 0),
    ((9, 7, 5), (3, 2, 2), 3),
    ((16, 16, 16), (2, 2, 2), 0),
    ((16, 16, 16), (2, 2, 2), 4),
    ((16, 16, 16), (4, 2, 2), 2),
    ((12, 10, 8), (1, 1, 1), 0),
    ((30, 20, 10), (3, 2, 1), 6),
    ((64, 32, 32), (4, 2, 2), 8),
]


def make_tables():
    exe = os.path.join(HERE, "_ref", "ref_tables_dump")
    subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True)
    out = []
    for g, p, r in TABLE_CASES:
        txt = subprocess.run([exe, *map(str, g), *map(str, p), str(r)], check=True,
                             capture_output=True, text=True).stdout
        d = json.loads(txt)
        out.append({"grid": g, "blocks_p": p, "ranks": r, **d})
    with open(os.path.join(GOLD, "ref_tables.json"), "w") as f:
        json.dump({"generator": "oracle/ref_tables_dump.cpp + reference proj/src/{grid,transfers,tables}.cpp",
                   "cases": out}, f, indent=0)


def make_sip():
    from oracle import oracle as O

    res = {}
    for name, kind, dims, prec, alpha, iters in [
        ("c0_small_f64", 0, (12, 10, 8), "f64", 0.92, 10),
        ("c0_small_f32", 0, (12, 10, 8), "f32", 0.92, 10),
        ("c2_small_f32", 2, (20, 12, 6), "f32", 0.92, 10),
        ("c0_alpha0_f64", 0, (9, 7, 5), "f64", 0.0, 6),
    ]:
        A = O.generate(kind, 1303 + kind, dims)
        phi = O.field(*dims)
        norms = O.solve(A, phi, alpha, iters, prec)
        res[name + "_norms"] = norms
        res[name + "_phi_sum"] = np.array([phi.sum(), np.abs(phi).sum()])
        res[name + "_phi_probe"] = phi[1:-1, 1:-1, 1:-1].ravel()[::17].copy()
    # two-block lattice (block-Jacobi), config-0 generator with per-block seed
    g, pd = (16, 10, 8), (2, 1, 1)
    origins, dims, nbr = O.lattice(g, pd)
    blocks = []
    for b in range(2):
        A = O.generate(0, 1303 + 3 + b, dims[b], g, origins[b])
        blocks.append((A, O.field(*dims[b])))
    norms, bn = O.solve_multi(blocks, nbr, 0.92, 8, "f64")
    res["multi2_norms"] = norms
    res["multi2_block_norms"] = bn
    res["multi2_phi_sum"] = np.array([sum(ph.sum() for _, ph in blocks)])
    np.savez(os.path.join(GOLD, "sip_golden.npz"), **res)


def make_perf():
    exe = os.path.join(HERE, "_ref", "ref_perf_dump")
    if not os.path.exists(exe):
        subprocess.run(["make", "-C", HERE, "ref"], check=True)
    with open(os.path.join(GOLD, "perf_scenarios.txt")) as f:
        out = subprocess.run([exe], stdin=f, capture_output=True, text=True, check=True).stdout
    with open(os.path.join(GOLD, "perf_golden.txt"), "w") as f:
        f.write(out)


if __name__ == "__main__":
    os.makedirs(GOLD, exist_ok=True)
    make_tables()
    make_sip()
    make_perf()
    print("golden fixtures written to", GOLD)
