"""GPU parity: CUDA SIP path (through the C-ABI) vs the CPU oracle.

Bar (BASELINE.json north_star): phi and per-iteration residual norms within
1e-12 relative (fp64) / 1e-5 relative (fp32).  Because every cell performs
the oracle's operations in the oracle's order (no FMA contraction), phi is
in fact expected BITWISE equal in both precisions; the norms differ only by
summation order (fp64 accumulation on both sides).
"""
import numpy as np
import pytest

import paper_1303_4538_b200 as sip
from oracle import oracle as O

pytestmark = pytest.mark.gpu

NORM_TOL = 1e-12


def _run_gpu(A, dims, prec, alpha, iters, phi0=None):
    s = sip.Solver(dims, prec)
    s.set_system(0, sip.StencilSystem.from_dict(A))
    s.factor(alpha)
    phi = O.field(*dims) if phi0 is None else phi0.copy()
    norms = s.solve([phi], iters)
    s.close()
    return phi, norms


def _run_oracle(A, dims, prec, alpha, iters, phi0=None):
    phi = O.field(*dims) if phi0 is None else phi0.copy()
    norms = O.solve(A, phi, alpha, iters, prec)
    return phi, norms


CASES = [
    # (dims, kind, iters) -- config 0 is (64,64,64), kind 0, 20 iterations
    ((64, 64, 64), 0, 20),
    ((37, 23, 19), 0, 6),      # ragged tiles in i and j
    ((16, 16, 40), 0, 5),      # exactly one tile, tall
    ((50, 33, 3), 0, 5),       # nz < tile skew
    ((2, 3, 2), 0, 4),         # tiny
    ((1, 2, 3), 0, 3),         # degenerate columns (nx = 1)
    ((40, 24, 20), 2, 6),      # config-2 generator (anisotropic convection-diffusion)
]


@pytest.mark.parametrize("prec", ["f64", "f32"])
@pytest.mark.parametrize("dims,kind,iters", CASES)
def test_solve_matches_oracle(gpu, dims, kind, iters, prec):
    A = O.generate(kind, 1303 + kind, dims)
    pg, ng = _run_gpu(A, dims, prec, 0.92, iters)
    po, no = _run_oracle(A, dims, prec, 0.92, iters)
    assert len(ng) == iters
    np.testing.assert_allclose(ng, no, rtol=NORM_TOL, atol=0)
    # bitwise phi (interior and untouched ghosts)
    assert np.array_equal(pg, po), f"max |diff| {np.abs(pg - po).max()}"


def test_nonzero_ghosts_and_phi0(gpu):
    """Dirichlet-style data in the ghost layer and a non-zero initial guess."""
    dims = (21, 18, 17)
    A = O.generate(0, 7, dims)
    # couple the boundary: make domain-boundary coefficients non-zero
    rng = np.random.default_rng(3)
    for n in ("AW", "AE", "AS", "AN", "AB", "AT"):
        A[n][1:-1, 1:-1, 1:-1] = np.where(A[n][1:-1, 1:-1, 1:-1] == 0.0, -0.7, A[n][1:-1, 1:-1, 1:-1])
    phi0 = rng.uniform(-1, 1, size=(dims[2] + 2, dims[1] + 2, dims[0] + 2))
    for prec in ("f64", "f32"):
        pg, ng = _run_gpu(A, dims, prec, 0.5, 5, phi0)
        po, no = _run_oracle(A, dims, prec, 0.5, 5, phi0)
        np.testing.assert_allclose(ng, no, rtol=NORM_TOL)
        assert np.array_equal(pg, po)


@pytest.mark.parametrize("alpha", [0.0, 0.5, 0.92])
def test_factor_alpha(gpu, alpha):
    dims = (30, 20, 10)
    A = O.generate(0, 11, dims)
    pg, ng = _run_gpu(A, dims, "f64", alpha, 3)
    po, no = _run_oracle(A, dims, "f64", alpha, 3)
    np.testing.assert_allclose(ng, no, rtol=NORM_TOL)
    assert np.array_equal(pg, po)


def test_singular_factor_names_cell(gpu):
    dims = (20, 20, 20)
    A = O.generate(0, 5, dims)
    A["AP"][7, 5, 9] = 0.0      # cell (i=9, j=5, k=7)
    A["AW"][7, 5, 9] = A["AE"][7, 5, 9] = A["AS"][7, 5, 9] = 0.0
    A["AN"][7, 5, 9] = A["AB"][7, 5, 9] = A["AT"][7, 5, 9] = 0.0
    A["AP"][3, 2, 4] = 0.0; A["AW"][3, 2, 4] = 0.0; A["AS"][3, 2, 4] = 0.0; A["AB"][3, 2, 4] = 0.0
    with pytest.raises(ValueError) as eo:
        O.factor(A, 0.0)
    s = sip.Solver(dims, "f64")
    s.set_system(0, sip.StencilSystem.from_dict(A))
    with pytest.raises(sip.SingularFactorError) as eg:
        s.factor(0.0)
    idx = int(str(eo.value).split()[-1])
    assert f"Field3 index {idx}" in str(eg.value)


def test_stale_and_misuse(gpu):
    dims = (10, 10, 10)
    A = O.generate(0, 1, dims)
    s = sip.Solver(dims, "f64")
    s.set_system(0, sip.StencilSystem.from_dict(A))
    with pytest.raises(sip.MisuseError):
        s.solve([O.field(*dims)], 2)
    s.factor(0.92)
    s.solve([O.field(*dims)], 2)
    s.set_system(0, sip.StencilSystem.from_dict(A))   # new revision
    with pytest.raises(sip.StaleFactorsError):
        s.solve([O.field(*dims)], 2)
    with pytest.raises(sip.ConfigError):
        s.factor(1.0)


def test_residual_general_matches_oracle(gpu):
    dims = (19, 17, 13)
    A = O.generate(0, 2, dims)
    rng = np.random.default_rng(0)
    fi = rng.uniform(-1, 1, size=(dims[2] + 2, dims[1] + 2, dims[0] + 2))
    rg = sip.residual_general(sip.StencilSystem.from_dict(A), fi)
    ro = O.residual(A, fi)
    assert np.array_equal(rg[1:-1, 1:-1, 1:-1], ro[1:-1, 1:-1, 1:-1])


def test_source_update_reuses_factors(gpu):
    """solve() on the reuse path: new su, same factors."""
    dims = (24, 24, 24)
    A = O.generate(0, 9, dims)
    S = sip.StencilSystem.from_dict(A)
    cfg = sip.SipConfig(alpha=0.92, max_iters=4)
    F = sip.sip_factor(S, cfg)
    n0 = sip.factorization_count()
    for seed in range(3):
        A2 = dict(A)
        A2["Q"] = O.generate(0, 100 + seed, dims)["Q"]
        S2 = sip.StencilSystem.from_dict(A2)
        fi, rep = sip.solve(S2, O.field(*dims), cfg, F)
        po = O.field(*dims)
        no = O.solve(A2, po, 0.92, 4)
        assert np.array_equal(fi, po)
        np.testing.assert_allclose(rep.norms, no, rtol=NORM_TOL)
    assert sip.factorization_count() == n0


def test_target_reduction(gpu):
    dims = (16, 16, 16)
    A = O.generate(0, 4, dims)
    S = sip.StencilSystem.from_dict(A)
    fi, rep = sip.solve(S, O.field(*dims), sip.SipConfig(max_iters=50, target=1.0))
    assert rep.iterations == 0 and np.all(fi == 0)
    fi, rep = sip.solve(S, O.field(*dims), sip.SipConfig(max_iters=200, target=1e-6))
    assert rep.norms[-1] / rep.norms[0] <= 1e-6
    assert rep.iterations < 200
