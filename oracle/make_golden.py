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
4. ftt1/ -- FTT1 transfer-table files written by the reference's own
   write_tables (build_transfer_tables over wall / periodic decompositions),
   their read-back entries (read_tables), and the reference reader's /
   validator's messages on deterministic corruptions of them
   (ftt1/cases.json); pins sip_ftt1_read / _write / _validate.
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


FTT1_CASES = [
    # name, gnx gny gnz, px py pz, ranks (0: one block per rank), periodic axis mask
    ("wall_2x2x1_r2", (16, 12, 8), (2, 2, 1), 2, 0),
    ("perx_2x2x1_r2", (16, 12, 8), (2, 2, 1), 2, 1),
    ("perall_2x1x1", (12, 12, 12), (2, 1, 1), 0, 7),
    ("peryz_1x2x2_r4", (8, 16, 16), (1, 2, 2), 0, 6),
    ("wall_3x1x2_r3", (17, 9, 10), (3, 1, 2), 3, 0),
    # single-rank tables (one GPU): table-driven halo vs the built-in plan / oracle
    ("wall_2x2x1_r1", (40, 36, 30), (2, 2, 1), 1, 0),
    ("perx_2x2x1_r1", (40, 36, 30), (2, 2, 1), 1, 1),
    ("perall_1x2x2_r1", (33, 20, 18), (1, 2, 2), 1, 7),
]

# corruptions of one base file: (name, base case, edit); edits are applied by
# tests/test_ftt1.py identically (ftt1_corrupt)
FTT1_CORRUPT = [
    ("trunc_magic", "perx_2x2x1_r2", ["truncate", 3]),
    ("trunc_version", "perx_2x2x1_r2", ["truncate", 6]),
    ("trunc_header", "perx_2x2x1_r2", ["truncate", 14]),
    ("trunc_count", "perx_2x2x1_r2", ["truncate", 18]),
    ("trunc_entry", "perx_2x2x1_r2", ["truncate", 20 + 40 + 17]),
    ("trunc_bounds", "perx_2x2x1_r2", ["truncate", 20 + 40 + 30]),
    ("bad_magic", "perx_2x2x1_r2", ["set", 1, 0x58]),
    ("bad_version", "perx_2x2x1_r2", ["set", 4, 2]),
    ("bad_dir", "perx_2x2x1_r2", ["set", 20 + 40, 3]),
    ("bad_kind", "perx_2x2x1_r2", ["set", 20 + 41, 7]),
    ("bad_face", "perx_2x2x1_r2", ["set", 20 + 42, 6]),
    # protocol: first entry of rank 1's table (a recv from rank 0) -> owner changed
    ("proto_owner", "wall_2x2x1_r2", ["set_u32_entry", 1, 0, 4, 3]),
    # rank 0's first send targets itself
    ("proto_self_send", "wall_2x2x1_r2", ["set_u32_entry", 0, 4, 3, 0]),
    # a local entry naming another rank as peer
    ("proto_local_peer", "wall_2x2x1_r2", ["set_u32_entry", 0, 0, 3, 1]),
    # cell-count mismatch: a recv's bounds widened
    ("proto_cells", "wall_2x2x1_r2", ["set_u32_entry", 1, 0, 7, 9]),
    # an orphan recv: rank 1's first entry turned into a recv from rank 2 (no sends from 2)
    ("proto_orphan", "wall_3x1x2_r3", ["set_u32_entry", 1, 0, 3, 2]),
]


def ftt1_corrupt(data: bytes, edit) -> bytes:
    """Apply one corruption recipe (shared with tests/test_ftt1.py)."""
    b = bytearray(data)
    if edit[0] == "truncate":
        return bytes(b[: edit[1]])
    if edit[0] == "set":
        b[edit[1]] = edit[2]
        return bytes(b)
    if edit[0] == "set_u32_entry":  # rank, entry index, u32 field index (3..11), value
        rank, k, field, val = edit[1:]
        off = 16
        for r in range(rank + 1):
            n = int.from_bytes(b[off:off + 4], "little")
            off += 4
            if r == rank:
                break
            off += 40 * n
        e = off + 40 * k
        fo = e + 4 + 4 * (field - 3)
        b[fo:fo + 4] = int(val).to_bytes(4, "little", signed=val < 0)
        return bytes(b)
    raise ValueError(edit)


def make_ftt1():
    exe = os.path.join(HERE, "_ref", "ref_ftt1_dump")
    if not os.path.exists(exe):
        subprocess.run(["make", "-C", HERE, "ref"], check=True)
    out = os.path.join(GOLD, "ftt1")
    os.makedirs(out, exist_ok=True)
    cases = {"generator": "oracle/ref_ftt1_dump.cpp + reference proj/src/{grid,transfers,tables}.cpp",
             "files": {}, "corrupt": {}}
    for name, g, p, ranks, mask in FTT1_CASES:
        path = os.path.join(out, name + ".ftt1")
        r = subprocess.run([exe, "make", *map(str, g), *map(str, p), str(ranks), str(mask), path],
                           capture_output=True, text=True, check=True).stdout
        cases["files"][name] = {"g": g, "p": p, "ranks": ranks, "periodic_mask": mask,
                                "entries": json.loads(r)["ranks"]}
    for name, base, edit in FTT1_CORRUPT:
        with open(os.path.join(out, base + ".ftt1"), "rb") as f:
            data = ftt1_corrupt(f.read(), edit)
        tmp = os.path.join(out, "_tmp.ftt1")
        with open(tmp, "wb") as f:
            f.write(data)
        rd = subprocess.run([exe, "read", tmp], capture_output=True, text=True, check=True).stdout.strip()
        va = subprocess.run([exe, "validate", tmp], capture_output=True, text=True, check=True).stdout.strip()
        os.remove(tmp)
        cases["corrupt"][name] = {"base": base, "edit": edit,
                                  "read": rd if rd.startswith("error: ") else "ok",
                                  "validate": va}
    with open(os.path.join(out, "cases.json"), "w") as f:
        json.dump(cases, f, indent=1)


if __name__ == "__main__":
    os.makedirs(GOLD, exist_ok=True)
    make_tables()
    make_sip()
    make_perf()
    make_ftt1()
    print("golden fixtures written to", GOLD)
