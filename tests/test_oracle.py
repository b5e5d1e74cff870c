"""CPU tests of the SIP oracle (oracle/sip_oracle.c): known-answer properties
from the reference specification, an independent numpy restatement, and the
committed golden vectors.  No GPU needed.

The reference has no SIP code, so the oracle is pinned by the
SPEC's own examples and properties:
  SPEC.md:149  pure diagonal system -> lp = 1/ap, other factors 0
  SPEC.md:150  alpha = 0: L*U reproduces A on the seven stencil positions
  SPEC.md:151  alpha > 0: corrected identity
  SPEC.md:158-160  fi = 0 -> res = su; residual matches a dense mat-vec
  SPEC.md:167  residual_symmetric == residual_general on symmetric systems
  SPEC.md:176  diagonal system converges in one sweep to su/ap
  SPEC.md:177, 194  residual non-increasing on SPD Poisson (alpha = 0)
  SPEC.md:178, 192  fp32 relaxation agrees with fp64 to 1e-4 once converged
  SPEC.md:186  manufactured solution: observed order >= 1.9
"""
import os

import numpy as np
import pytest

from oracle import oracle as O
from oracle import oracle_np as N

GOLD = os.path.join(os.path.dirname(__file__), "golden")
NB = {"W": (0, 0, -1), "E": (0, 0, 1), "S": (0, -1, 0), "N": (0, 1, 0), "B": (-1, 0, 0), "T": (1, 0, 0)}


def interior(a):
    return a[1:-1, 1:-1, 1:-1]


def dense_from(A, which=("AW", "AE", "AS", "AN", "AB", "AT"), diag="AP"):
    """Dense matrix of the 7-point system over interior cells (lexicographic)."""
    nz, ny, nx = (s - 2 for s in A[diag].shape)
    n = nx * ny * nz
    idx = lambda i, j, k: i + nx * (j + ny * k)
    M = np.zeros((n, n))
    for k in range(nz):
        for j in range(ny):
            for i in range(nx):
                r = idx(i, j, k)
                M[r, r] = A[diag][k + 1, j + 1, i + 1]
                for name in which:
                    dk, dj, di = NB[name[1]]
                    ii, jj, kk = i + di, j + dj, k + dk
                    if 0 <= ii < nx and 0 <= jj < ny and 0 <= kk < nz:
                        M[r, idx(ii, jj, kk)] = A[name][k + 1, j + 1, i + 1]
    return M


def lu_dense(F, dims):
    """Dense L (diag 1/LP, LW/LS/LB) and U (unit diag, UN/UE/UT)."""
    nx, ny, nz = dims
    n = nx * ny * nz
    idx = lambda i, j, k: i + nx * (j + ny * k)
    L = np.zeros((n, n))
    U = np.eye(n)
    for k in range(nz):
        for j in range(ny):
            for i in range(nx):
                r = idx(i, j, k)
                c = (k + 1, j + 1, i + 1)
                L[r, r] = 1.0 / F["LP"][c]
                if i > 0: L[r, idx(i - 1, j, k)] = F["LW"][c]
                if j > 0: L[r, idx(i, j - 1, k)] = F["LS"][c]
                if k > 0: L[r, idx(i, j, k - 1)] = F["LB"][c]
                if i < nx - 1: U[r, idx(i + 1, j, k)] = F["UE"][c]
                if j < ny - 1: U[r, idx(i, j + 1, k)] = F["UN"][c]
                if k < nz - 1: U[r, idx(i, j, k + 1)] = F["UT"][c]
    return L, U


def random_system(dims, seed, symmetric=False):
    rng = np.random.default_rng(seed)
    nx, ny, nz = dims
    A = {n: O.field(*dims) for n in O.ARRAYS}
    for n in ("AW", "AE", "AS", "AN", "AB", "AT"):
        interior(A[n])[...] = -rng.uniform(0.5, 1.5, size=(nz, ny, nx))
    if symmetric:
        # A_W(i) = A_E(i-1) etc.
        interior(A["AW"])[:, :, 1:] = interior(A["AE"])[:, :, :-1]
        interior(A["AS"])[:, 1:, :] = interior(A["AN"])[:, :-1, :]
        interior(A["AB"])[1:, :, :] = interior(A["AT"])[:-1, :, :]
    interior(A["AW"])[:, :, 0] = 0; interior(A["AE"])[:, :, -1] = 0
    interior(A["AS"])[:, 0, :] = 0; interior(A["AN"])[:, -1, :] = 0
    interior(A["AB"])[0, :, :] = 0; interior(A["AT"])[-1, :, :] = 0
    s = sum(np.abs(A[n]) for n in ("AW", "AE", "AS", "AN", "AB", "AT"))
    A["AP"][...] = 1.05 * s
    interior(A["Q"])[...] = rng.uniform(-1, 1, size=(nz, ny, nx))
    return A


# --------------------------------------------------------------- restatements
@pytest.mark.parametrize("dims", [(5, 4, 3), (3, 6, 4), (7, 2, 5), (1, 3, 2)])
@pytest.mark.parametrize("alpha", [0.0, 0.5, 0.92])
def test_c_oracle_matches_numpy_restatement(dims, alpha):
    A = O.generate(0, 1303, dims)
    F = O.factor(A, alpha)
    Fn = N.factor(A, alpha)
    for n in F:
        assert np.array_equal(F[n], Fn[n]), n
    p1, p2 = O.field(*dims), O.field(*dims)
    for _ in range(3):
        a, b = O.sweep(A, F, p1), N.sweep(A, Fn, p2)
        assert np.array_equal(p1, p2)
        assert a == pytest.approx(b, rel=1e-14)
    # fp32 relaxation arrays
    A32 = {n: v.astype(np.float32) for n, v in A.items()}
    F32 = {n: v.astype(np.float32) for n, v in F.items()}
    q1, q2 = O.field(*dims, np.float32), O.field(*dims, np.float32)
    for _ in range(3):
        a, b = O.sweep(A32, F32, q1), N.sweep(A32, F32, q2)
        assert np.array_equal(q1, q2)
        assert a == pytest.approx(b, rel=1e-14)


def test_generator_matches_library_generator():
    import paper_1303_4538_b200 as sip
    for kind in (0, 2):
        for dims, g, o in [((6, 5, 4), None, (0, 0, 0)), ((4, 3, 2), (9, 7, 5), (4, 2, 3))]:
            A = O.generate(kind, 1303 + kind, dims, g, o)
            B = sip.generate_host(kind, 1303 + kind, dims, g, o)
            for n in O.ARRAYS:
                assert np.array_equal(A[n], B[n]), (kind, n)


def test_generator_zeroes_domain_boundary_and_dominance():
    A = O.generate(0, 7, (6, 5, 4))
    assert np.all(A["AW"][1:-1, 1:-1, 1] == 0) and np.all(A["AE"][1:-1, 1:-1, -2] == 0)
    assert np.all(A["AS"][1:-1, 1, 1:-1] == 0) and np.all(A["AN"][1:-1, -2, 1:-1] == 0)
    assert np.all(A["AB"][1, 1:-1, 1:-1] == 0) and np.all(A["AT"][-2, 1:-1, 1:-1] == 0)
    s = sum(np.abs(interior(A[n])) for n in ("AW", "AE", "AS", "AN", "AB", "AT"))
    assert np.allclose(interior(A["AP"]), 1.01 * s, rtol=1e-15)
    assert np.all(interior(A["Q"]) >= -1) and np.all(interior(A["Q"]) < 1)


# --------------------------------------------------------------- SPEC KATs
def test_diagonal_system_one_sweep():
    dims = (4, 3, 5)
    A = {n: O.field(*dims) for n in O.ARRAYS}
    rng = np.random.default_rng(1)
    interior(A["AP"])[...] = rng.uniform(1, 3, size=(5, 3, 4))
    interior(A["Q"])[...] = rng.uniform(-1, 1, size=(5, 3, 4))
    F = O.factor(A, 0.92)
    assert np.array_equal(interior(F["LP"]), 1.0 / interior(A["AP"]))
    for n in ("LB", "LW", "LS", "UN", "UE", "UT"):
        assert not np.any(F[n])
    phi = O.field(*dims)
    n0 = O.sweep(A, F, phi)
    assert n0 == pytest.approx(np.abs(interior(A["Q"])).sum(), rel=1e-15)   # fi = 0 -> res = su
    assert np.allclose(interior(phi), interior(A["Q"]) / interior(A["AP"]), rtol=1e-15)
    n1 = O.sweep(A, F, phi)
    assert n1 <= 1e-15 * n0


def test_first_norm_is_sum_abs_q():
    dims = (8, 7, 6)
    A = O.generate(0, 3, dims)
    norms = O.solve(A, O.field(*dims), 0.92, 2)
    assert norms[0] == pytest.approx(np.abs(interior(A["Q"])).sum(), rel=1e-13)


@pytest.mark.parametrize("dims", [(3, 3, 3), (4, 3, 2)])
def test_lu_identity_alpha0(dims):
    A = random_system(dims, 11, symmetric=True)
    F = O.factor(A, 0.0)
    Lm, Um = lu_dense(F, dims)
    M = dense_from(A)
    LU = Lm @ Um
    stencil = M != 0
    np.fill_diagonal(stencil, True)
    assert np.max(np.abs((LU - M)[stencil])) < 1e-12


@pytest.mark.parametrize("alpha", [0.5, 0.92])
def test_lu_identity_alpha_corrected(alpha):
    """SPEC.md:151 claims LU == A on the stencil for alpha > 0; that is false for
    Stone's recurrence.  The exact identity:
      (LU)_P = AP+P1+P2+P3, (LU)_N = AN-P1, (LU)_E = AE-P2, (LU)_T = AT-P3,
      (LU)_W = AW - a*LW(UN_W+UT_W), (LU)_S = AS - a*LS(UE_S+UT_S),
      (LU)_B = AB - a*LB(UN_B+UE_B), plus fill LW*UN_W, LW*UT_W, LS*UE_S,
      LS*UT_S, LB*UN_B, LB*UE_B."""
    dims = (4, 3, 3)
    A = random_system(dims, 5)
    F = O.factor(A, alpha)
    Lm, Um = lu_dense(F, dims)
    LU = Lm @ Um
    nx, ny, nz = dims
    idx = lambda i, j, k: i + nx * (j + ny * k)
    g = lambda a, i, j, k: a[k + 1, j + 1, i + 1] if 0 <= i < nx and 0 <= j < ny and 0 <= k < nz else 0.0
    for k in range(nz):
        for j in range(ny):
            for i in range(nx):
                r = idx(i, j, k)
                unB, ueB = g(F["UN"], i, j, k - 1), g(F["UE"], i, j, k - 1)
                unW, utW = g(F["UN"], i - 1, j, k), g(F["UT"], i - 1, j, k)
                ueS, utS = g(F["UE"], i, j - 1, k), g(F["UT"], i, j - 1, k)
                lb, lw, ls = g(F["LB"], i, j, k), g(F["LW"], i, j, k), g(F["LS"], i, j, k)
                p1 = alpha * (lb * unB + lw * unW)
                p2 = alpha * (lb * ueB + ls * ueS)
                p3 = alpha * (lw * utW + ls * utS)
                exp = {r: g(A["AP"], i, j, k) + p1 + p2 + p3}
                if i + 1 < nx: exp[idx(i + 1, j, k)] = g(A["AE"], i, j, k) - p2
                if j + 1 < ny: exp[idx(i, j + 1, k)] = g(A["AN"], i, j, k) - p1
                if k + 1 < nz: exp[idx(i, j, k + 1)] = g(A["AT"], i, j, k) - p3
                if i > 0: exp[idx(i - 1, j, k)] = g(A["AW"], i, j, k) - alpha * lw * (unW + utW)
                if j > 0: exp[idx(i, j - 1, k)] = g(A["AS"], i, j, k) - alpha * ls * (ueS + utS)
                if k > 0: exp[idx(i, j, k - 1)] = g(A["AB"], i, j, k) - alpha * lb * (unB + ueB)
                # fill entries
                if i > 0 and j + 1 < ny: exp[idx(i - 1, j + 1, k)] = lw * unW
                if i > 0 and k + 1 < nz: exp[idx(i - 1, j, k + 1)] = lw * utW
                if j > 0 and i + 1 < nx: exp[idx(i + 1, j - 1, k)] = ls * ueS
                if j > 0 and k + 1 < nz: exp[idx(i, j - 1, k + 1)] = ls * utS
                if k > 0 and j + 1 < ny: exp[idx(i, j + 1, k - 1)] = lb * unB
                if k > 0 and i + 1 < nx: exp[idx(i + 1, j, k - 1)] = lb * ueB
                row = np.zeros(LU.shape[1])
                for c, v in exp.items():
                    row[c] = v
                assert np.max(np.abs(LU[r] - row)) < 1e-12


def test_residual_matches_dense_matvec():
    dims = (4, 4, 3)
    A = random_system(dims, 2)
    rng = np.random.default_rng(9)
    fi = O.field(*dims)
    interior(fi)[...] = rng.uniform(-1, 1, size=(3, 4, 4))
    res = O.residual(A, fi)
    M = dense_from(A)
    ref = interior(A["Q"]).ravel() - M @ interior(fi).ravel()
    assert np.max(np.abs(interior(res).ravel() - ref)) < 1e-13
    assert np.array_equal(interior(O.residual(A, O.field(*dims))), interior(A["Q"]))


def test_residual_symmetric_equals_general():
    dims = (5, 4, 3)
    A = random_system(dims, 4, symmetric=True)
    rng = np.random.default_rng(2)
    fi = rng.uniform(-1, 1, size=A["AP"].shape)
    rg = O.residual(A, fi)
    rs = O.residual_symmetric(A, fi)
    assert np.max(np.abs(interior(rg) - interior(rs))) <= 1e-15


def poisson(n, h=None):
    """Uniform 7-point Laplacian on an n^3 unit cube with homogeneous Dirichlet
    boundaries folded into AP (matrix-entry signs), manufactured source."""
    h = h or 1.0 / n
    A = {k: O.field(n, n, n) for k in O.ARRAYS}
    for name in ("AW", "AE", "AS", "AN", "AB", "AT"):
        interior(A[name])[...] = -1.0
    interior(A["AW"])[:, :, 0] = 0; interior(A["AE"])[:, :, -1] = 0
    interior(A["AS"])[:, 0, :] = 0; interior(A["AN"])[:, -1, :] = 0
    interior(A["AB"])[0, :, :] = 0; interior(A["AT"])[-1, :, :] = 0
    # Dirichlet walls at distance h/2: ghost = -phi -> AP += 1 per boundary face
    interior(A["AP"])[...] = 6.0
    interior(A["AP"])[:, :, 0] += 1; interior(A["AP"])[:, :, -1] += 1
    interior(A["AP"])[:, 0, :] += 1; interior(A["AP"])[:, -1, :] += 1
    interior(A["AP"])[0, :, :] += 1; interior(A["AP"])[-1, :, :] += 1
    x = (np.arange(n) + 0.5) * h
    Z, Y, X = np.meshgrid(x, x, x, indexing="ij")
    exact = np.sin(np.pi * X) * np.sin(np.pi * Y) * np.sin(np.pi * Z)
    interior(A["Q"])[...] = 3 * np.pi ** 2 * exact * h * h
    return A, exact


def test_monotone_residual_poisson_alpha0():
    A, _ = poisson(8)
    norms = O.solve(A, O.field(8, 8, 8), 0.0, 10)
    assert np.all(np.diff(norms) <= 0)


def test_manufactured_solution_order():
    errs = []
    for n in (8, 16, 32):
        A, exact = poisson(n)
        phi = O.field(n, n, n)
        O.solve(A, phi, 0.92, 400)
        errs.append(np.max(np.abs(interior(phi) - exact)))
    orders = [np.log2(errs[i] / errs[i + 1]) for i in range(2)]
    assert min(orders) >= 1.9, (errs, orders)


def test_fp32_relaxation_agrees_with_fp64():
    A, _ = poisson(12)
    p64, p32 = O.field(12, 12, 12), O.field(12, 12, 12)
    n64 = O.solve(A, p64, 0.92, 200)
    n32 = O.solve(A, p32, 0.92, 200, "f32")
    assert n64[-1] / n64[0] < 1e-6
    assert np.max(np.abs(p32 - p64)) / np.max(np.abs(p64)) <= 1e-4


def test_singular_factor_names_first_cell():
    A = O.generate(0, 5, (6, 5, 4))
    for n in O.ARRAYS[:7]:
        A[n][3, 2, 4] = 0.0
        A[n][2, 4, 1] = 0.0
    with pytest.raises(ValueError) as e:
        O.factor(A, 0.92)
    # first in lexicographic (k, j, i) order: cell (i=1, j=4, k=2)
    assert int(str(e.value).split()[-1]) == 1 + 8 * (4 + 7 * 2)


# --------------------------------------------------------------- golden vectors
def test_golden_vectors():
    g = np.load(os.path.join(GOLD, "sip_golden.npz"))
    for name, kind, dims, prec, alpha, iters in [
        ("c0_small_f64", 0, (12, 10, 8), "f64", 0.92, 10),
        ("c0_small_f32", 0, (12, 10, 8), "f32", 0.92, 10),
        ("c2_small_f32", 2, (20, 12, 6), "f32", 0.92, 10),
        ("c0_alpha0_f64", 0, (9, 7, 5), "f64", 0.0, 6),
    ]:
        A = O.generate(kind, 1303 + kind, dims)
        phi = O.field(*dims)
        norms = O.solve(A, phi, alpha, iters, prec)
        assert np.array_equal(norms, g[name + "_norms"]), name
        assert np.array_equal(interior(phi).ravel()[::17], g[name + "_phi_probe"]), name


def test_multiblock_block_jacobi():
    g, pd = (16, 10, 8), (2, 1, 1)
    origins, dims, nbr = O.lattice(g, pd)
    blocks = [(O.generate(0, 1303 + 3 + b, dims[b], g, origins[b]), O.field(*dims[b]))
              for b in range(2)]
    norms, bn = O.solve_multi(blocks, nbr, 0.92, 8, "f64")
    gold = np.load(os.path.join(GOLD, "sip_golden.npz"))
    assert np.array_equal(norms, gold["multi2_norms"])
    assert np.array_equal(bn, gold["multi2_block_norms"])
    assert np.allclose(norms, bn.sum(axis=1), rtol=1e-15)
    # threaded relaxation of the blocks gives identical results
    blocks2 = [(O.generate(0, 1303 + 3 + b, dims[b], g, origins[b]), O.field(*dims[b]))
               for b in range(2)]
    norms2, _ = O.solve_multi(blocks2, nbr, 0.92, 8, "f64", nthreads=2)
    assert np.array_equal(norms, norms2)
    for (_, a), (_, b) in zip(blocks, blocks2):
        assert np.array_equal(a, b)


def test_multiblock_single_block_equals_solve():
    dims = (10, 9, 7)
    A = O.generate(0, 1303, dims)
    p1 = O.field(*dims)
    n1 = O.solve(A, p1, 0.92, 5)
    p2 = O.field(*dims)
    n2, _ = O.solve_multi([(A, p2)], [(-1,) * 6], 0.92, 5)
    assert np.array_equal(p1, p2) and np.array_equal(n1, n2)


def test_lattice_matches_reference_decompose():
    import json
    with open(os.path.join(GOLD, "ref_tables.json")) as f:
        cases = json.load(f)["cases"]
    for c in cases:
        origins, dims, _ = O.lattice(c["grid"], c["blocks_p"])
        for b, (lo0, lo1, lo2, hi0, hi1, hi2, _) in enumerate(c["blocks"]):
            assert origins[b] == (lo0, lo1, lo2)
            assert dims[b] == (hi0 - lo0 + 1, hi1 - lo1 + 1, hi2 - lo2 + 1)


def test_symmetric_generator_invariant():
    """Generator kind 3: AW(i) = AE(i-1), AS(j) = AN(j-1), AB(k) = AT(k-1)
    exactly, boundary-pointing coefficients zero; Listing-1
    residual equals the general one bitwise."""
    dims = (9, 7, 6)
    A = O.generate(3, 5, dims)
    I = (slice(1, -1),) * 3
    assert np.array_equal(A["AW"][1:-1, 1:-1, 2:-1], A["AE"][1:-1, 1:-1, 1:-2])
    assert np.array_equal(A["AS"][1:-1, 2:-1, 1:-1], A["AN"][1:-1, 1:-2, 1:-1])
    assert np.array_equal(A["AB"][2:-1, 1:-1, 1:-1], A["AT"][1:-2, 1:-1, 1:-1])
    assert not A["AW"][1:-1, 1:-1, 1].any() and not A["AE"][1:-1, 1:-1, -2].any()
    fi = np.random.default_rng(3).uniform(-1, 1, size=A["AP"].shape)
    assert np.array_equal(O.residual_symmetric(A, fi)[I], O.residual(A, fi)[I])


@pytest.mark.parametrize("prec", ["f64", "f32"])
@pytest.mark.parametrize("nthreads", [1, 2, 3, 7, 64])
def test_pipelined_sweep_matches_serial(prec, nthreads):
    """The multi-threaded oracle sweep (the CPU reference arm of bench.py) is
    bitwise equal to the serial sweep in phi; norms to 1e-12."""
    dims = (13, 11, 9)
    A = O.generate(0, 1303, dims)
    F = O.factor(A, 0.92)
    dt = np.float64 if prec == "f64" else np.float32
    A = {n: v.astype(dt) for n, v in A.items()}
    F = {n: v.astype(dt) for n, v in F.items()}
    p1 = O.field(*dims, dtype=dt)
    p2 = O.field(*dims, dtype=dt)
    work = O.field(*dims, dtype=dt)
    for _ in range(3):
        n1 = O.sweep(A, F, p1)
        n2 = O.sweep_pipe(A, F, p2, nthreads, work)
        assert np.array_equal(p1, p2)
        assert n2 == pytest.approx(n1, rel=1e-12)


@pytest.mark.parametrize("prec", ["f64", "f32"])
def test_solve_pipe_equals_solve(prec):
    """solve_pipe (factor + threaded sweeps, the full-size parity driver) is
    bitwise the serial orc_solve; the norms are summed per thread (1e-12)."""
    dims = (21, 35, 9)
    A = O.generate(0, 77, dims)
    p1, p2 = O.field(*dims), O.field(*dims)
    p1[0, :, :] = 0.3  # a B ghost plane: kept by both
    p2[0, :, :] = 0.3
    n1 = O.solve(A, p1, 0.92, 6, prec)
    n2 = O.solve_pipe(A, p2, 0.92, 6, prec, nthreads=4)
    assert np.array_equal(p1, p2)
    np.testing.assert_allclose(n1, n2, rtol=1e-12, atol=0)


@pytest.mark.parametrize("prec", ["f64", "f32"])
def test_solve_multi_gen_equals_solve_multi(prec):
    """The memory-lean block-Jacobi driver (systems regenerated per iteration)
    gives orc_solve_multi's phi and block norms bit for bit."""
    g, pd = (30, 26, 20), (3, 2, 2)
    origins, dims, nbr = O.lattice(g, pd)
    blocks = [(O.generate(0, 500 + b, dims[b], g, origins[b]), O.field(*dims[b])) for b in range(len(dims))]
    n1, b1 = O.solve_multi(blocks, nbr, 0.92, 5, prec, nthreads=3)
    phis = [O.field(*d) for d in dims]
    n2, b2 = O.solve_multi_gen(0, 500, g, pd, phis, 0.92, 5, prec, nthreads=3)
    np.testing.assert_array_equal(b1, b2)
    np.testing.assert_array_equal(n1, n2)
    for (A, p), q in zip(blocks, phis):
        assert np.array_equal(p, q)
