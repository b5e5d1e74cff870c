"""Multi-rank block-Jacobi SIP on CPU (gloo, world_size 2): exercises the
library's host-side halo plan (sip_plan_halo / sip_plan_block_ranks) the way
its NCCL path uses it -- per peer, send entries packed in plan order, receive
entries unpacked in plan order (one ncclSend / ncclRecv pair per peer) --
with the CPU oracle doing the per-block sweeps.  The result must be bitwise
identical to the single-process block-Jacobi oracle (decomposition-invariant
coupling, SPEC.md:364 / SURVEY.md 8c item 8)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

G, PD, ITERS, ALPHA = (16, 10, 8), (2, 2, 1), 6, 0.92


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _box(phi, e):
    ilo, ihi, jlo, jhi, klo, khi = e[6:12]
    return (slice(klo, khi + 1), slice(jlo, jhi + 1), slice(ilo, ihi + 1))


def _periodic_system(A, d, o, g, mask):
    """Restore the couplings across periodic boundaries (as the GPU test)."""
    A = {n: a.copy() for n, a in A.items()}
    inner = (slice(1, -1),) * 3
    for axis, (lo_arr, hi_arr) in enumerate((("AW", "AE"), ("AS", "AN"), ("AB", "AT"))):
        if not (mask >> axis) & 1:
            continue
        sl_lo, sl_hi = [slice(1, -1)] * 3, [slice(1, -1)] * 3
        sl_lo[2 - axis], sl_hi[2 - axis] = slice(1, 2), slice(-2, -1)
        if o[axis] == 0:
            A[lo_arr][tuple(sl_lo)] = -0.75
        if o[axis] + d[axis] == g[axis]:
            A[hi_arr][tuple(sl_hi)] = -0.75
    A["AP"][inner] = 1.01 * sum(np.abs(A[n][inner]) for n in ("AW", "AE", "AS", "AN", "AB", "AT"))
    return A


def _system(O, b, dims, origins, g, mask):
    A = O.generate(0, 1303 + 3 + b, dims[b], g, origins[b])
    return _periodic_system(A, dims[b], origins[b], g, mask) if mask else A


def _worker(rank, world, port, out, case=None):
    import sys
    sys.path.insert(0, ROOT)
    import paper_1303_4538_b200 as sip
    from oracle import oracle as O

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g, pd, mask = (G, PD, 0) if case is None else (case["g"], case["p"], case["mask"])
    origins, dims, nbr = O.lattice(g, pd)
    if case is None:
        br = sip.plan_block_ranks(pd, world)
        plan = sip.plan_halo(g, pd, br, rank).tolist()
    else:  # reference-written FTT1 table: block placement and plan from the file
        tables = sip.ftt1_read(open(case["file"], "rb").read())
        br = [0] * len(dims)
        for r, t in enumerate(tables):
            for row in t.tolist():
                if row[0] != 2:
                    br[row[4]] = r
        plan = [row for row in tables[rank].tolist() if row[1] == 0]
    mine = [b for b in range(len(dims)) if br[b] == rank]
    A = {b: _system(O, b, dims, origins, g, mask) for b in mine}
    F = {b: O.factor(A[b], ALPHA) for b in mine}
    phi = {b: O.field(*dims[b]) for b in mine}
    peers = sorted({e[3] for e in plan if e[0] != 0})

    def exchange():
        for e in plan:  # local copies: owner = src block, neighbor = dst block
            if e[0] == 0:
                src, dst = e[4], e[5]
                face = e[2] ^ 1  # ghost face on the destination (opposite)
                dbox = _ghost_box(dims[dst], face)
                phi[dst][dbox] = phi[src][_box(phi[src], e)]
        reqs, bufs = [], {}
        for q in peers:
            sends = [phi[e[4]][_box(phi[e[4]], e)].ravel() for e in plan if e[0] == 1 and e[3] == q]
            rsz = sum(int(np.prod(phi[e[4]][_box(phi[e[4]], e)].shape)) for e in plan
                      if e[0] == 2 and e[3] == q)
            bufs[q] = torch.zeros(rsz, dtype=torch.float64)
            reqs.append(dist.irecv(bufs[q], src=q))
            reqs.append(dist.isend(torch.from_numpy(np.concatenate(sends)), dst=q))
        for r in reqs:
            r.wait()
        for q in peers:
            off = 0
            for e in plan:
                if e[0] == 2 and e[3] == q:
                    box = _box(phi[e[4]], e)
                    n = int(np.prod(phi[e[4]][box].shape))
                    phi[e[4]][box] = bufs[q][off:off + n].numpy().reshape(phi[e[4]][box].shape)
                    off += n

    exchange()
    norms = []
    for _ in range(ITERS):
        bn = np.zeros(len(dims))
        for b in mine:
            bn[b] = O.sweep(A[b], F[b], phi[b])
        t = torch.from_numpy(bn)
        dist.all_reduce(t)  # disjoint blocks: the sum is an all-gather
        norms.append(float(sum(t.numpy())))  # block-id order, as the library
        exchange()
    out[rank] = {"norms": norms, "phi": {b: phi[b] for b in mine}}
    dist.destroy_process_group()


def _ghost_box(d, face):
    nx, ny, nz = d
    full = {0: (nx + 1, nx + 1, 1, ny, 1, nz), 1: (0, 0, 1, ny, 1, nz),
            2: (1, nx, ny + 1, ny + 1, 1, nz), 3: (1, nx, 0, 0, 1, nz),
            4: (1, nx, 1, ny, nz + 1, nz + 1), 5: (1, nx, 1, ny, 0, 0)}[face]
    ilo, ihi, jlo, jhi, klo, khi = full
    return (slice(klo, khi + 1), slice(jlo, jhi + 1), slice(ilo, ihi + 1))


def _wrap(nbr, pd, mask):
    px, py, pz = pd
    out = []
    for b, n in enumerate(nbr):
        c = [b % px, (b // px) % py, b // (px * py)]
        n = list(n)
        for axis in range(3):
            if (mask >> axis) & 1:
                for s, slot in ((-1, 2 * axis), (1, 2 * axis + 1)):
                    q = list(c)
                    q[axis] = (q[axis] + s) % pd[axis]
                    n[slot] = q[0] + px * (q[1] + py * q[2])
        out.append(tuple(n))
    return out


@pytest.mark.parametrize("source", ["plan_halo", "ftt1_periodic"])
def test_two_rank_block_jacobi_matches_single_process(source):
    from oracle import oracle as O
    world = 2
    case = None
    g, pd, mask = G, PD, 0
    if source == "ftt1_periodic":  # reference-written table, periodic in x, 2 ranks
        import json
        gold = os.path.join(ROOT, "tests", "golden", "ftt1")
        f = json.load(open(os.path.join(gold, "cases.json")))["files"]["perx_2x2x1_r2"]
        g, pd, mask = tuple(f["g"]), tuple(f["p"]), f["periodic_mask"]
        case = {"g": g, "p": pd, "mask": mask, "file": os.path.join(gold, "perx_2x2x1_r2.ftt1")}
    mgr = mp.Manager()
    out = mgr.dict()
    mp.start_processes(_worker, args=(world, _port(), out, case), nprocs=world, join=True,
                       start_method="spawn")
    origins, dims, nbr = O.lattice(g, pd)
    blocks = [(_system(O, b, dims, origins, g, mask), O.field(*dims[b])) for b in range(len(dims))]
    ref_norms, _ = O.solve_multi(blocks, _wrap(nbr, pd, mask), ALPHA, ITERS, "f64")
    for r in range(world):
        np.testing.assert_allclose(out[r]["norms"], ref_norms, rtol=1e-14)
        for b, ph in out[r]["phi"].items():
            assert np.array_equal(ph[1:-1, 1:-1, 1:-1], blocks[b][1][1:-1, 1:-1, 1:-1]), b
