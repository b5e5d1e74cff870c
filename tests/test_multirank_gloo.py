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


def _worker(rank, world, port, out):
    import sys
    sys.path.insert(0, ROOT)
    import paper_1303_4538_b200 as sip
    from oracle import oracle as O

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    origins, dims, nbr = O.lattice(G, PD)
    br = sip.plan_block_ranks(PD, world)
    mine = [b for b in range(len(dims)) if br[b] == rank]
    A = {b: O.generate(0, 1303 + 3 + b, dims[b], G, origins[b]) for b in mine}
    F = {b: O.factor(A[b], ALPHA) for b in mine}
    phi = {b: O.field(*dims[b]) for b in mine}
    plan = sip.plan_halo(G, PD, br, rank).tolist()
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


def test_two_rank_block_jacobi_matches_single_process():
    from oracle import oracle as O
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.start_processes(_worker, args=(world, _port(), out), nprocs=world, join=True,
                       start_method="spawn")
    origins, dims, nbr = O.lattice(G, PD)
    blocks = [(O.generate(0, 1303 + 3 + b, dims[b], G, origins[b]), O.field(*dims[b]))
              for b in range(len(dims))]
    ref_norms, _ = O.solve_multi(blocks, nbr, ALPHA, ITERS, "f64")
    for r in range(world):
        np.testing.assert_allclose(out[r]["norms"], ref_norms, rtol=1e-14)
        for b, ph in out[r]["phi"].items():
            assert np.array_equal(ph[1:-1, 1:-1, 1:-1], blocks[b][1][1:-1, 1:-1, 1:-1]), b
