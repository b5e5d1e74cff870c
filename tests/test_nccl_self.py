"""The multi-rank exchange path on real hardware with one GPU.

With SIPB_NCCL_SELF=1 a single-rank context routes every local face
transfer through the inter-GPU path -- per-peer pack kernels, ncclSend /
ncclRecv inside one group (here to the rank itself), unpack kernels -- so the
NCCL code that a multi-GPU run executes (sip_api.cu exchange(), sip_flow.cu
flow_exchange()) is exercised and checked bitwise against the block-Jacobi
oracle.  (A second GPU is not available to this test-suite; the multi-rank
host logic is covered by tests/test_multirank_gloo.py.)
"""
import os

import numpy as np
import pytest

import paper_1303_4538_b200 as sip
from oracle import flow as OF
from oracle import oracle as O


@pytest.fixture
def nccl_self():
    old = os.environ.get("SIPB_NCCL_SELF")
    os.environ["SIPB_NCCL_SELF"] = "1"
    yield
    if old is None:
        del os.environ["SIPB_NCCL_SELF"]
    else:
        os.environ["SIPB_NCCL_SELF"] = old


@pytest.mark.gpu
@pytest.mark.parametrize("prec", ["f64", "f32"])
def test_sip_through_nccl_matches_oracle(gpu, nccl_self, prec):
    g, pd = (40, 36, 24), (2, 2, 2)
    iters = 5
    s = sip.Solver(None, prec, 0, lattice=(g, pd))
    origins, dims, nbr = O.lattice(g, pd)
    As = []
    for lb, (bid, d, o) in enumerate(s.blocks):
        A = O.generate(0, 1303 + 9 + bid, d, g, o)
        As.append(A)
        s.set_system(lb, sip.StencilSystem.from_dict(A))
    s.factor(0.92)
    phis = [O.field(*d) for (_, d, _) in s.blocks]
    s.load_phi(phis)
    s.iterate(iters)
    ng = s.read_norms(0, iters)
    launches = s.launch_count()
    s.store_phi(phis)
    s.close()
    blocks = [(As[b], O.field(*dims[b])) for b in range(8)]
    no, _ = O.solve_multi(blocks, nbr, 0.92, iters, prec)
    np.testing.assert_allclose(ng, no, rtol=1e-12)
    for b in range(8):
        assert np.array_equal(phis[b], blocks[b][1]), f"block {b}"
    # the self mode really took the pack / NCCL / unpack path: one unpack
    # launch per exchange on top of the copy / pack launch
    os.environ["SIPB_NCCL_SELF"] = "0"
    s2 = sip.Solver(None, prec, 0, lattice=(g, pd))
    for lb in range(len(s2.blocks)):
        s2.set_system(lb, sip.StencilSystem.from_dict(As[lb]))
    s2.factor(0.92)
    s2.load_phi([O.field(*d) for (_, d, _) in s2.blocks])
    s2.iterate(iters)
    plain = s2.launch_count()
    s2.close()
    assert launches == plain + (iters + 1), (launches, plain)


@pytest.mark.gpu
def test_pressure_correct_through_nccl_matches_oracle(gpu, nccl_self):
    from test_flow import _smooth_fields  # noqa: E402  (tests/ is on sys.path)
    g, pd, bc = (16, 12, 8), (2, 2, 1), (OF.PERIODIC, OF.PERIODIC, OF.WALL, OF.WALL, OF.WALL, OF.WALL)
    lengths, dt, cap, sweeps = (1.0, 0.75, 0.5), 0.05, 2, 3
    s = sip.Solver(None, "f64", 0, lattice=(g, pd))
    s.assemble_poisson(lengths, ("periodic", "periodic", "wall", "wall", "wall", "wall"))
    s.factor(0.92)
    us, vs, ws, ps = _smooth_fields(g, pd)
    fl = sip.Flow(s)
    bids = [bid for (bid, _, _) in s.blocks]
    for name, arrs in zip("uvwp", (us, vs, ws, ps)):
        fl.set(name, [arrs[b] for b in bids])
    with pytest.raises(sip.NonConvergenceError):
        fl.pressure_correct(dt, 0.0, cap, sweeps)
    got = {}
    for name in "uvwp":
        arrs = [O.field(*d) for (_, d, _) in s.blocks]
        fl.get(name, arrs)
        got[name] = arrs
    fl.close()
    s.close()
    As = OF.assemble_poisson(g, pd, lengths, bc)
    _, _, nbr = OF.wrapped_lattice(g, pd, bc)
    with pytest.raises(RuntimeError):
        OF.pressure_correct(As, nbr, us, vs, ws, ps, OF.cell_sizes(g, lengths), dt, 0.0, cap, sweeps)
    for name, ref in zip("uvwp", (us, vs, ws, ps)):
        for lb, bid in enumerate(bids):
            assert np.array_equal(got[name][lb][(slice(1, -1),) * 3], ref[bid][(slice(1, -1),) * 3]), (name, bid)
