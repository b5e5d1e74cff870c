"""The split face-halo exchange.

With SIPB_XSPLIT=1 a multi-block context runs the exchange in two phases:
the copies / packs whose source is an E, N or T interior plane start on a
comm stream as soon as K2 has finished. They wait on K3's per-brick stamps,
so they run while K3 is still sweeping. The rest follows K3. The default
(SIPB_XSPLIT unset / 0) is the single stream-ordered exchange after K3
(measured as fast or faster on one GPU). Both must give the block-Jacobi
oracle's phi bitwise. The split mode launches one extra kernel per iteration
(early and late copies separately).
"""
import os

import numpy as np
import pytest

import paper_1303_4538_b200 as sip
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _run(g, pd, prec, iters, seed, split, nccl_self=False, graph=False, calls=1):
    env = {"SIPB_XSPLIT": "1" if split else "0", "SIPB_NCCL_SELF": "1" if nccl_self else "0",
           "SIPB_GRAPH": "1" if graph else "0"}
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        s = sip.Solver(None, prec, 0, lattice=(g, pd))
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    As = []
    for lb, (bid, d, o) in enumerate(s.blocks):
        A = O.generate(0, seed + bid, d, g, o)
        As.append(A)
        s.set_system(lb, sip.StencilSystem.from_dict(A))
    s.factor(0.92)
    phis = [O.field(*d) for (_, d, _) in s.blocks]
    s.load_phi(phis)
    for _ in range(calls):
        s.iterate(iters)
    iters *= calls
    norms = s.read_norms(0, iters)
    launches = s.launch_count()
    s.store_phi(phis)
    s.close()
    return As, phis, norms, launches


def _oracle(As, g, pd, prec, iters):
    _, dims, nbr = O.lattice(g, pd)
    blocks = [(As[b], O.field(*dims[b])) for b in range(len(As))]
    no, _ = O.solve_multi(blocks, nbr, 0.92, iters, prec)
    return [b[1] for b in blocks], no


@pytest.mark.parametrize("prec", ["f64", "f32"])
def test_split_exchange_matches_oracle(gpu, prec):
    g, pd, iters = (40, 36, 24), (2, 2, 2), 6
    As, phis, ng, l_split = _run(g, pd, prec, iters, 1303 + 40, True)
    po, no = _oracle(As, g, pd, prec, iters)
    np.testing.assert_allclose(ng, no, rtol=1e-12)
    for b in range(len(po)):
        assert np.array_equal(phis[b], po[b]), f"block {b}"
    _, phis0, ng0, l_plain = _run(g, pd, prec, iters, 1303 + 40, False)
    assert np.array_equal(np.asarray(ng0), np.asarray(ng))
    for b in range(len(po)):
        assert np.array_equal(phis0[b], po[b]), f"block {b} (unsplit)"
    assert l_split == l_plain + iters, (l_split, l_plain)


@pytest.mark.parametrize("prec", ["f64", "f32"])
def test_split_exchange_many_blocks_many_iterations(gpu, prec):
    """A 4x3x2 lattice of uneven blocks (partial bricks on every side) over
    20 iterations: each iteration's early copies race K3 on the same blocks;
    any copy that ran before its plane was final would show as a phi mismatch."""
    g, pd, iters = (92, 70, 30), (4, 3, 2), 20
    As, phis, ng, _ = _run(g, pd, prec, iters, 1303 + 60, True)
    po, no = _oracle(As, g, pd, prec, iters)
    np.testing.assert_allclose(ng, no, rtol=1e-12)
    for b in range(len(po)):
        assert np.array_equal(phis[b], po[b]), f"block {b}"


def test_split_exchange_through_nccl(gpu):
    """Split mode with every transfer through NCCL (self-exchange): phase 1
    sends the early planes during K3, phase 2 the rest; four exchange
    launches per iteration instead of two."""
    g, pd, iters = (40, 36, 24), (2, 2, 2), 5
    As, phis, ng, l_self = _run(g, pd, "f64", iters, 1303 + 80, True, nccl_self=True)
    po, no = _oracle(As, g, pd, "f64", iters)
    np.testing.assert_allclose(ng, no, rtol=1e-12)
    for b in range(len(po)):
        assert np.array_equal(phis[b], po[b]), f"block {b}"
    _, _, _, l_plain = _run(g, pd, "f64", iters, 1303 + 80, True)
    # initial exchange (unsplit): +1 unpack launch; per iteration: +2 (early
    # and late unpacks)
    assert l_self == l_plain + 2 * iters + 1, (l_self, l_plain)


def test_split_exchange_in_cuda_graph(gpu):
    """SIPB_GRAPH=1 with the split exchange: the capture forks to the comm
    stream (ev_k2, ev_k3) and joins back (ev_x); replayed three times."""
    g, pd, iters = (40, 24, 20), (2, 1, 1), 2
    As, phis, ng, _ = _run(g, pd, "f64", iters, 1303 + 90, True, graph=True, calls=3)
    po, no = _oracle(As, g, pd, "f64", 3 * iters)
    np.testing.assert_allclose(ng, no, rtol=1e-12)
    for b in range(len(po)):
        assert np.array_equal(phis[b], po[b]), f"block {b}"
