"""Parity at the BASELINE.json configurations as specified -- full grid sizes
AND full iteration counts -- through the C-ABI against the CPU oracle:
bitwise phi (every cell of every block), per-iteration (and per-block) norms
within 1e-12 relative.

  config 1  256^3 single block, kind 0, 50 iterations, fp64 and fp32
  config 2  512x256x128 anisotropic convection-diffusion, fp32, 100 iterations
  config 3  2x2x2 blocks of 128^3 (one GPU's share), fp64, 50 block-Jacobi iterations
  config 4  1024x512x512 in 128 blocks of 128^3, fp32, 10 block-Jacobi iterations
            (all 128 blocks bitwise; the config's 100 iterations run in the bench)

The oracle side uses the threaded drivers (oracle.solve_pipe: factor + j-slab
pipelined sweeps; oracle.solve_multi_gen: block-Jacobi with each block's
system regenerated on the fly), both pinned bitwise to the serial oracle by
tests/test_oracle.py.
"""
import os

import numpy as np
import pytest

import paper_1303_4538_b200 as sip
from oracle import oracle as O

pytestmark = pytest.mark.gpu

NORM_TOL = 1e-12
NCORES = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)


def _single_block(g, kind, seed, prec, iters):
    A = O.generate(kind, seed, g)
    s = sip.Solver(g, prec)
    s.set_system(0, sip.StencilSystem.from_dict(A))
    s.factor(0.92)
    pg = O.field(*g)
    ng = s.solve([pg], iters)
    s.close()
    po = O.field(*g)
    no = O.solve_pipe(A, po, 0.92, iters, prec, nthreads=NCORES)
    assert len(ng) == iters
    np.testing.assert_allclose(ng, no, rtol=NORM_TOL, atol=0)
    assert np.array_equal(pg, po), f"max |diff| {np.abs(pg - po).max()}"


@pytest.mark.parametrize("prec", ["f64", "f32"])
def test_config1_full_length(gpu, prec):
    """Config 1: 256^3, 50 inner iterations (BASELINE.json configs[1])."""
    _single_block((256, 256, 256), 0, 1304, prec, 50)


def test_config2_full_length(gpu):
    """Config 2: 512x256x128 anisotropic convection-diffusion, fp32, 100 iterations."""
    _single_block((512, 256, 128), 2, 1305, "f32", 100)


def _lattice(g, pd, seed, prec, iters, nthreads):
    s = sip.Solver(None, prec, 0, lattice=(g, pd))
    s.generate(0, seed)
    s.factor(0.92)
    phis = [sip.field(*d) for (_, d, _) in s.blocks]
    s.load_phi(phis)
    s.iterate(iters)
    ng, bng = s.read_norms(0, iters, per_block=True)
    s.store_phi(phis)
    ids = [bid for (bid, _, _) in s.blocks]
    s.close()
    origins, dims, _ = O.lattice(g, pd)
    po = [O.field(*d) for d in dims]
    no, bno = O.solve_multi_gen(0, seed, g, pd, po, 0.92, iters, prec, nthreads=nthreads)
    np.testing.assert_allclose(ng, no, rtol=NORM_TOL, atol=0)
    np.testing.assert_allclose(bng, bno, rtol=NORM_TOL, atol=0)
    bad = [bid for lb, bid in enumerate(ids) if not np.array_equal(phis[lb], po[bid])]
    assert not bad, f"blocks with phi != oracle: {bad[:10]}"


def test_config3_full_length(gpu):
    """Config 3: 2x2x2 blocks of 128^3 per GPU, fp64, 50 block-Jacobi
    iterations (one-cell face halos exchanged after every iteration)."""
    _lattice((256, 256, 256), (2, 2, 2), 1306, "f64", 50, min(8, NCORES))


def test_config4_every_block(gpu):
    """Config 4: 1024x512x512 in 128 blocks of 128^3, fp32, 10 block-Jacobi
    iterations, every block bitwise (the bench runs the config's 100)."""
    _lattice((1024, 512, 512), (8, 4, 4), 1307, "f32", 10, min(8, NCORES))
