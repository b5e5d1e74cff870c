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
    # (dims, kind, iters) -- config 0 is (64,64,64), kind 0, 20 iterations; bricks are
    # 8 (i) x 32 (j) columns
    ((64, 64, 64), 0, 20),
    ((37, 23, 19), 0, 6),      # ragged bricks in i and j
    ((16, 16, 40), 0, 5),      # tall, half a brick in j
    ((50, 33, 3), 0, 5),       # nz < brick skew
    ((2, 3, 2), 0, 4),         # tiny
    ((1, 2, 3), 0, 3),         # degenerate columns (nx = 1)
    ((40, 24, 20), 2, 6),      # config-2 generator (anisotropic convection-diffusion)
    ((8, 32, 16), 0, 5),       # exactly one brick: E and N ghosts in ghost bricks
    ((24, 96, 5), 0, 4),       # exact 3 x 3 bricks
    ((9, 33, 7), 0, 4),        # one-cell-wide second brick in i and in j
    ((16, 64, 1), 0, 4),       # nz = 1
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


@pytest.mark.parametrize("prec", ["f64", "f32"])
def test_single_cell(gpu, prec):
    """A 1x1x1 grid.  The generator's single cell has every coupling on the
    domain boundary, so AP = 0: both the library and the oracle reject it,
    naming the same cell.  With AP set and the boundary coupled (Dirichlet
    ghosts) the one-cell solve is bitwise equal to the oracle."""
    dims = (1, 1, 1)
    A = O.generate(0, 1303, dims)
    with pytest.raises(sip.SingularFactorError, match="Field3 index 13"):
        _run_gpu(A, dims, prec, 0.92, 3)
    with pytest.raises(ValueError, match="Field3 index 13"):
        _run_oracle(A, dims, prec, 0.92, 3)
    for n, v in (("AW", -0.5), ("AE", -0.25), ("AS", -0.125), ("AN", -0.75), ("AB", -0.3), ("AT", -0.6)):
        A[n][1, 1, 1] = v
    A["AP"][1, 1, 1] = 3.5
    phi0 = np.random.default_rng(5).uniform(-1, 1, size=(3, 3, 3))
    pg, ng = _run_gpu(A, dims, prec, 0.92, 4, phi0)
    po, no = _run_oracle(A, dims, prec, 0.92, 4, phi0)
    np.testing.assert_allclose(ng, no, rtol=NORM_TOL, atol=0)
    assert np.array_equal(pg, po)


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


def _symmetrize(A):
    """A_W(i) = A_E(i-1), A_S(j) = A_N(j-1), A_B(k) = A_T(k-1) over the whole
    Field3 (ghost layers included), so the SPEC.md:117 invariant holds."""
    S = {n: a.copy() for n, a in A.items()}
    S["AW"][:, :, 1:] = S["AE"][:, :, :-1]
    S["AS"][:, 1:, :] = S["AN"][:, :-1, :]
    S["AB"][1:, :, :] = S["AT"][:-1, :, :]
    return S


@pytest.mark.parametrize("dims", [(19, 17, 13), (40, 33, 20), (1, 5, 4)])
def test_residual_symmetric_matches_oracle(gpu, dims):
    """residual_symmetric (Listing 1) on the device, bitwise
    vs the oracle's Listing-1 restatement and vs residual_general."""
    A = _symmetrize(O.generate(0, 5, dims))
    rng = np.random.default_rng(1)
    fi = rng.uniform(-1, 1, size=(dims[2] + 2, dims[1] + 2, dims[0] + 2))
    S = sip.StencilSystem.from_dict(A, symmetric=True)
    rs = sip.residual_symmetric(S, fi)
    ro = O.residual_symmetric(A, fi)
    rg = sip.residual_general(S, fi)
    inner = (slice(1, -1),) * 3
    assert np.array_equal(rs[inner], ro[inner])
    assert np.array_equal(rs[inner], rg[inner])


def test_residual_symmetric_errors(gpu):
    dims = (12, 10, 8)
    A = O.generate(0, 6, dims)
    fi = O.field(*dims)
    with pytest.raises(sip.MisuseError):  # not flagged
        sip.residual_symmetric(sip.StencilSystem.from_dict(A), fi)
    with pytest.raises(sip.ConfigError):  # flagged, but the coefficients are not symmetric
        sip.residual_symmetric(sip.StencilSystem.from_dict(A, symmetric=True), fi)
    s = sip.Solver(dims, "f64")
    s.set_system(0, sip.StencilSystem.from_dict(_symmetrize(A)))
    s.set_symmetric(0, True)
    s.load_phi([fi])
    s.residual(symmetric=True)
    s.set_system(0, sip.StencilSystem.from_dict(_symmetrize(A)))  # new revision clears the flag
    with pytest.raises(sip.MisuseError):
        s.residual(symmetric=True)
    s.close()


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


@pytest.mark.parametrize("prec", ["f64", "f32"])
@pytest.mark.parametrize("g,pd", [((40, 36, 30), (2, 2, 2)), ((33, 17, 20), (3, 1, 2)),
                                  ((64, 48, 32), (2, 3, 1)),
                                  ((32, 128, 16), (2, 2, 2))])  # brick-exact blocks: E/N ghost bricks
def test_multiblock_matches_oracle(gpu, g, pd, prec):
    """Block-structured lattice on one GPU: per-block factorisation, one-cell
    face halos exchanged after every inner iteration (device copies), norms
    summed in block order -- identical to the block-Jacobi oracle."""
    iters = 6
    s = sip.Solver(None, prec, 0, lattice=(g, pd))
    origins, dims, nbr = O.lattice(g, pd)
    assert [d for (_, d, _) in s.blocks] == [tuple(x) for x in dims]
    As = []
    for lb, (bid, d, o) in enumerate(s.blocks):
        A = O.generate(0, 1303 + 3 + bid, d, g, o)
        As.append(A)
        s.set_system(lb, sip.StencilSystem.from_dict(A))
    s.factor(0.92)
    phis = [O.field(*d) for (_, d, _) in s.blocks]
    s.load_phi(phis)
    s.iterate(iters)
    ng, bng = s.read_norms(0, iters, per_block=True)
    s.store_phi(phis)
    s.close()
    blocks = [(As[b], O.field(*dims[b])) for b in range(len(dims))]
    no, bno = O.solve_multi(blocks, nbr, 0.92, iters, prec)
    np.testing.assert_allclose(ng, no, rtol=NORM_TOL)
    np.testing.assert_allclose(bng, bno, rtol=NORM_TOL)
    for b in range(len(dims)):
        assert np.array_equal(phis[b], blocks[b][1]), f"block {b}"


def test_device_generator_matches_host(gpu):
    g, pd = (30, 20, 12), (2, 2, 1)
    s = sip.Solver(None, "f64", 0, lattice=(g, pd))
    s.generate(0, 99)
    s.factor(0.92)
    phis = [O.field(*d) for (_, d, _) in s.blocks]
    s.load_phi(phis)
    s.iterate(3)
    ng = s.read_norms(0, 3)
    s.close()
    origins, dims, nbr = O.lattice(g, pd)
    blocks = [(O.generate(0, 99 + b, dims[b], g, origins[b]), O.field(*dims[b])) for b in range(4)]
    no, _ = O.solve_multi(blocks, nbr, 0.92, 3, "f64")
    np.testing.assert_allclose(ng, no, rtol=NORM_TOL)


def test_config1_full_size_properties(gpu):
    """Config 1 (256^3, fp64) at full size: residual norms decrease, the first
    norm equals sum|Q| (phi0 = 0), and the GPU residual of the final phi agrees
    with the last+1 norm (checksum of checksums)."""
    g = (256, 256, 256)
    s = sip.Solver(None, "f64", 0, lattice=(g, (1, 1, 1)))
    s.generate(0, 1304)
    s.factor(0.92)
    s.load_phi([sip.field(*g)])
    s.iterate(12)
    n = s.read_norms(0, 12)
    res = s.residual()[0]
    s.close()
    A = O.generate(0, 1304, g)
    assert n[0] == pytest.approx(np.abs(A["Q"]).sum(), rel=1e-12)
    assert np.all(np.diff(n) < 0)
    # residual of the phi after 12 iterations == the (unrun) 13th pre-update norm
    r13 = np.abs(res[1:-1, 1:-1, 1:-1]).sum()
    assert r13 < n[-1]


def _periodic_system(A, d, o, g, mask):
    """Generator system of one block with the couplings across periodic
    domain boundaries restored (the generator zeroes every boundary-pointing
    coefficient) and AP re-balanced: 1.01 * sum |A_nb|."""
    A = {n: a.copy() for n, a in A.items()}
    inner = (slice(1, -1),) * 3
    for axis, (lo_arr, hi_arr) in enumerate((("AW", "AE"), ("AS", "AN"), ("AB", "AT"))):
        if not (mask >> axis) & 1:
            continue
        sl_lo = [slice(1, -1)] * 3
        sl_hi = [slice(1, -1)] * 3
        ax = 2 - axis  # Field3 arrays are (k, j, i)
        sl_lo[ax] = slice(1, 2)
        sl_hi[ax] = slice(-2, -1)
        if o[axis] == 0:
            A[lo_arr][tuple(sl_lo)] = -0.75
        if o[axis] + d[axis] == g[axis]:
            A[hi_arr][tuple(sl_hi)] = -0.75
    s = sum(np.abs(A[n][inner]) for n in ("AW", "AE", "AS", "AN", "AB", "AT"))
    A["AP"][inner] = 1.01 * s
    return A


@pytest.mark.parametrize("prec", ["f64", "f32"])
@pytest.mark.parametrize("name", ["wall_2x2x1_r1", "perx_2x2x1_r1", "perall_1x2x2_r1"])
def test_table_driven_halo_matches_oracle(gpu, name, prec):
    """Face halos driven by an FTT1 table written by the reference
    (tests/golden/ftt1/, periodic wraps included, px = 1 self-wrap in
    perall_1x2x2): bitwise equal to the block-Jacobi oracle with the same
    (wrapped) neighbour table."""
    import json
    import os
    gold = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "ftt1")
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
        for axis, (c, p_) in enumerate(((bx, px), (by, py), (bz, pz))):
            if (mask >> axis) & 1:
                lo = [bx, by, bz]; hi = [bx, by, bz]
                lo[axis] -= 1; hi[axis] += 1
                n[2 * axis], n[2 * axis + 1] = bid(*lo), bid(*hi)
        wrapped.append(tuple(n))
    iters = 6
    s = sip.Solver(None, prec, 0, lattice=(g, pd))
    As = []
    for lb, (bid_, d, o) in enumerate(s.blocks):
        A = _periodic_system(O.generate(0, 1303 + 7 + bid_, d, g, o), d, o, g, mask)
        As.append(A)
        s.set_system(lb, sip.StencilSystem.from_dict(A))
    s.set_halo_tables(tables)
    s.factor(0.92)
    phis = [O.field(*d) for (_, d, _) in s.blocks]
    s.load_phi(phis)
    s.iterate(iters)
    ng = s.read_norms(0, iters)
    s.store_phi(phis)
    s.close()
    blocks = [(As[b], O.field(*dims[b])) for b in range(len(dims))]
    no, _ = O.solve_multi(blocks, wrapped, 0.92, iters, prec)
    np.testing.assert_allclose(ng, no, rtol=NORM_TOL)
    for b in range(len(dims)):
        assert np.array_equal(phis[b], blocks[b][1]), f"block {b}"


def test_halo_tables_rejects_bad_tables(gpu):
    import json
    import os
    gold = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "ftt1")
    f = json.load(open(os.path.join(gold, "cases.json")))["files"]["wall_2x2x1_r1"]
    tables = sip.ftt1_read(open(os.path.join(gold, "wall_2x2x1_r1.ftt1"), "rb").read())
    s = sip.Solver(None, "f64", 0, lattice=(tuple(f["g"]), tuple(f["p"])))
    bad = [t.copy() for t in tables]
    bad[0][0, 3] = 1  # a local entry naming another rank
    with pytest.raises(sip.ProtocolError):
        s.set_halo_tables(bad)
    with pytest.raises(sip.ConfigError):  # a 2-rank table set on a 1-rank context
        s.set_halo_tables(tables + [tables[0][:0]])
    part = [t.copy() for t in tables]
    face_rows = np.where(part[0][:, 1] == 0)[0]
    part[0][face_rows[0], 9] -= 1  # shrink the first face patch
    with pytest.raises(sip.ConfigError):
        s.set_halo_tables(part)
    s.close()


# ------------------------------------------------ SURVEY 8(c) known answers on the device
def test_kat_diagonal_system_converges_in_one_sweep(gpu):
    """KAT 1: a pure diagonal system gives LP = 1/AP and the
    first sweep lands on Q/AP exactly; the next residual norm is 0."""
    dims = (20, 18, 17)
    A = O.generate(0, 21, dims)
    for n in ("AW", "AE", "AS", "AN", "AB", "AT"):
        A[n][...] = 0.0
    s = sip.Solver(dims, "f64")
    s.set_system(0, sip.StencilSystem.from_dict(A))
    s.factor(0.92)
    phi = O.field(*dims)
    norms = s.solve([phi], 2)
    s.close()
    inner = (slice(1, -1),) * 3
    assert np.array_equal(phi[inner], A["Q"][inner] / A["AP"][inner] * 1.0) or \
        np.allclose(phi[inner], A["Q"][inner] / A["AP"][inner], rtol=1e-15, atol=0)
    assert norms[1] <= 1e-14 * norms[0]


@pytest.mark.parametrize("prec", ["f64", "f32"])
def test_kat_first_norm_is_sum_abs_q(gpu, prec):
    """KAT 2: phi0 = 0 -> residual = su -> norm[0] = sum |Q|."""
    dims = (33, 29, 21)
    A = O.generate(2, 22, dims)
    s = sip.Solver(dims, prec)
    s.set_system(0, sip.StencilSystem.from_dict(A))
    s.factor(0.92)
    n = s.solve([O.field(*dims)], 1)
    s.close()
    q = A["Q"][1:-1, 1:-1, 1:-1]
    ref = np.abs(q).sum() if prec == "f64" else np.abs(q.astype(np.float32).astype(np.float64)).sum()
    assert n[0] == pytest.approx(ref, rel=1e-12)


def test_kat_fp32_fp64_agree_when_converged(gpu):
    """KAT 7: fp32 and fp64 solutions agree to <= 1e-4 relative
    once converged."""
    dims = (24, 24, 24)
    A = O.generate(0, 23, dims)
    out = {}
    for prec in ("f64", "f32"):
        s = sip.Solver(dims, prec)
        s.set_system(0, sip.StencilSystem.from_dict(A))
        s.factor(0.92)
        phi = O.field(*dims)
        s.solve([phi], 200)
        s.close()
        out[prec] = phi[1:-1, 1:-1, 1:-1]
    rel = np.abs(out["f32"] - out["f64"]).max() / np.abs(out["f64"]).max()
    assert rel <= 1e-4


def test_kat_decomposition_independent_of_placement(gpu):
    """KAT 8: block-Jacobi coupling does not depend on where a
    block lives -- the same lattice solved with the library's compact
    placement and with the reference's with_ranks placement (one rank here)
    gives bitwise the same norms and phi."""
    g, pd = (32, 24, 20), (2, 2, 1)
    res = []
    for br in (None, [0, 0, 0, 0]):
        s = sip.Solver(None, "f64", 0, lattice=(g, pd), block_rank=br)
        for lb, (bid, d, o) in enumerate(s.blocks):
            s.set_system(lb, sip.StencilSystem.from_dict(O.generate(0, 1303 + 3 + bid, d, g, o)))
        s.factor(0.92)
        phis = [O.field(*d) for (_, d, _) in s.blocks]
        s.load_phi(phis)
        s.iterate(5)
        n = s.read_norms(0, 5)
        s.store_phi(phis)
        s.close()
        res.append((n, phis))
    assert np.array_equal(res[0][0], res[1][0])
    for a, b in zip(res[0][1], res[1][1]):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("prec", ["f64", "f32"])
@pytest.mark.parametrize("g,pd", [((37, 23, 19), (1, 1, 1)), ((40, 36, 30), (2, 2, 1)),
                                  ((33, 17, 20), (3, 1, 2))])
def test_symmetric_sweep_fast_path(gpu, g, pd, prec):
    """a system flagged symmetric runs K2's Listing-1 fast
    path (AW/AS/AB read as the neighbours' AE/AN/AT, 11 instead of 14 array
    touches per cell); phi bitwise equal to the oracle's general sweep."""
    iters = 5
    s = sip.Solver(None, prec, 0, lattice=(g, pd))
    origins, dims, nbr = O.lattice(g, pd)
    As = []
    for lb, (bid, d, o) in enumerate(s.blocks):
        A = _symmetrize(O.generate(0, 1303 + 11 + bid, d, g, o))
        As.append(A)
        s.set_system(lb, sip.StencilSystem.from_dict(A))
        s.set_symmetric(lb, True)
    s.factor(0.92)
    phis = [O.field(*d) for (_, d, _) in s.blocks]
    s.load_phi(phis)
    s.iterate(iters)
    ng = s.read_norms(0, iters)
    s.store_phi(phis)
    s.close()
    blocks = [(As[b], O.field(*dims[b])) for b in range(len(dims))]
    no, _ = O.solve_multi(blocks, nbr, 0.92, iters, prec)
    np.testing.assert_allclose(ng, no, rtol=NORM_TOL)
    for b in range(len(dims)):
        assert np.array_equal(phis[b], blocks[b][1]), f"block {b}"


def test_symmetric_generator_and_fast_path(gpu):
    """Device kind-3 (symmetric) generator == oracle generator; the device
    invariant check accepts it; the flagged fast path matches the oracle."""
    dims = (30, 22, 18)
    s = sip.Solver(None, "f64", 0, lattice=(dims, (1, 1, 1)))
    s.generate(3, 77)
    s.set_symmetric(0, True)
    s.factor(0.92)
    phi = O.field(*dims)
    s.load_phi([phi])
    s.iterate(4)
    n = s.read_norms(0, 4)
    s.store_phi([phi])
    s.close()
    A = O.generate(3, 77, dims)
    po = O.field(*dims)
    no = O.solve(A, po, 0.92, 4, "f64")
    np.testing.assert_allclose(n, no, rtol=NORM_TOL)
    assert np.array_equal(phi, po)


@pytest.mark.parametrize("prec", ["f64", "f32"])
def test_cuda_graph_replay_matches_oracle(gpu, prec):
    """sip_iterate through a captured CUDA graph (SIPB_GRAPH=1; replayed for
    every call with the same iteration count, norm slots from the device
    counter) gives the oracle's phi bitwise and its norms."""
    import os
    old = os.environ.get("SIPB_GRAPH")
    os.environ["SIPB_GRAPH"] = "1"
    try:
        g, pd = (40, 24, 20), (2, 1, 1)
        s = sip.Solver(None, prec, 0, lattice=(g, pd))
        origins, dims, nbr = O.lattice(g, pd)
        As = []
        for lb, (bid, d, o) in enumerate(s.blocks):
            A = O.generate(0, 1303 + 21 + bid, d, g, o)
            As.append(A)
            s.set_system(lb, sip.StencilSystem.from_dict(A))
        s.factor(0.92)
        phis = [O.field(*d) for (_, d, _) in s.blocks]
        s.load_phi(phis)
        for _ in range(3):
            s.iterate(2)  # capture once, replay twice
        ng = s.read_norms(0, 6)
        s.store_phi(phis)
        s.close()
    finally:
        if old is None:
            del os.environ["SIPB_GRAPH"]
        else:
            os.environ["SIPB_GRAPH"] = old
    blocks = [(As[b], O.field(*dims[b])) for b in range(2)]
    no, _ = O.solve_multi(blocks, nbr, 0.92, 6, prec)
    np.testing.assert_allclose(ng, no, rtol=NORM_TOL)
    for b in range(2):
        assert np.array_equal(phis[b], blocks[b][1])


@pytest.mark.parametrize("check_every", [1, 3, 8, 0])
@pytest.mark.parametrize("prec", ["f64", "f32"])
def test_target_mode_stops_exactly_on_device(gpu, prec, check_every):
    """Target reduction with the norm-evaluation interval:
    the forward sweep's finaliser tests norm / norm[0] <= target on the
    device, so the solve runs exactly the sweeps up to the first one meeting
    the target whatever the host poll interval; phi bitwise = the oracle run
    for that many sweeps."""
    dims = (24, 20, 18)
    A = O.generate(0, 91, dims)
    target = 1e-5
    s = sip.Solver(dims, prec)
    s.set_system(0, sip.StencilSystem.from_dict(A))
    s.factor(0.92)
    pg = O.field(*dims)
    ng = s.solve([pg], 300, target, check_every=check_every)
    s.close()
    # the oracle's stopping sweep
    full = O.solve(A, O.field(*dims), 0.92, 300, prec)
    want = next(i + 1 for i in range(300) if full[i] / full[0] <= target)
    assert len(ng) == want
    po = O.field(*dims)
    no = O.solve(A, po, 0.92, want, prec)
    np.testing.assert_allclose(ng, no, rtol=NORM_TOL, atol=0)
    assert np.array_equal(pg, po)


def test_target_mode_multiblock_and_reuse(gpu):
    """Device stop on a block lattice, then a fixed-count solve on the same
    context (the stop flag is reset per solve); library factor counter = 1."""
    g, pd = (40, 36, 30), (2, 2, 1)
    s = sip.Solver(None, "f64", 0, lattice=(g, pd))
    s.generate(0, 1306)
    s.factor(0.92)
    phis = [O.field(*d) for (_, d, _) in s.blocks]
    n1 = s.solve(phis, 400, 1e-4, check_every=5)
    assert 1 < len(n1) < 400 and n1[-1] / n1[0] <= 1e-4 and n1[-2] / n1[0] > 1e-4
    phis = [O.field(*d) for (_, d, _) in s.blocks]
    n2 = s.solve(phis, 7)
    assert len(n2) == 7
    np.testing.assert_array_equal(n2, n1[:7])
    assert s.factor_count() == 1
    s.factor(0.5)
    assert s.factor_count() == 2
    s.close()


@pytest.mark.parametrize("prec", ["f64", "f32"])
def test_async_pipeline_equals_sequential(gpu, prec):
    """sip_set_source_async / sip_solve_async (the next step's source uploaded
    while the current solve runs) give the sequential calls' phi and norms
    bit for bit, with a different source every step and phi0 = the previous
    step's result."""
    dims, iters, steps = (37, 29, 21), 4, 4
    A = O.generate(0, 1303 + 70, dims)
    rng = np.random.default_rng(9)
    qs = [A["Q"] * (1.0 + 0.25 * k) + rng.uniform(-0.1, 0.1, size=A["Q"].shape) for k in range(steps)]
    for q in qs:
        q[0, :, :] = q[-1, :, :] = 0.0  # ghosts of Q are not read; keep them tidy

    def make():
        s = sip.Solver(dims, prec)
        s.set_system(0, sip.StencilSystem.from_dict(A))
        s.factor(0.92)
        return s

    s = make()
    phi = O.field(*dims)
    seq_phi, seq_n = [], []
    for q in qs:
        s.set_source(0, q)
        seq_n.append(np.asarray(s.solve([phi], iters)))
        seq_phi.append(phi.copy())
    s.close()

    s = make()
    phi = O.field(*dims)
    s.set_source_async(0, qs[0])
    for k in range(steps):
        norms = np.zeros(iters)
        s.solve_async([phi], iters, norms)
        if k + 1 < steps:
            s.set_source_async(0, qs[k + 1])
        s.synchronize()
        assert np.array_equal(norms, seq_n[k]), k
        assert np.array_equal(phi, seq_phi[k]), k
    s.close()


def test_two_async_solves_in_flight(gpu):
    """The bench's e2e pattern: two solves pending, the next step's phi0 upload
    following the previous result's download chunk by chunk (same buffers),
    the next source uploaded during the current solve; bitwise equal to the
    sequential calls."""
    dims, iters, steps = (33, 40, 17), 3, 5
    A = O.generate(0, 1303 + 71, dims)
    qs = [A["Q"] * (1.0 + 0.125 * k) for k in range(steps)]

    def make():
        s = sip.Solver(dims, "f64")
        s.set_system(0, sip.StencilSystem.from_dict(A))
        s.factor(0.92)
        return s

    s = make()
    phi = O.field(*dims)
    seq_phi, seq_n = [], []
    for q in qs:
        s.set_source(0, q)
        seq_n.append(np.asarray(s.solve([phi], iters)))
        seq_phi.append(phi.copy())
    s.close()

    s = make()
    phi = O.field(*dims)
    norms = [np.zeros(iters) for _ in range(steps)]
    s.set_source_async(0, qs[0])
    s.solve_async([phi], iters, norms[0])
    for k in range(steps):
        if k + 1 < steps:
            s.set_source_async(0, qs[k + 1])
            s.solve_async([phi], iters, norms[k + 1])
        s.wait_async()
        assert np.array_equal(norms[k], seq_n[k]), k
        if k + 1 == steps:
            assert np.array_equal(phi, seq_phi[k])
    s.synchronize()
    s.close()


def test_two_async_solves_multiblock(gpu):
    """Two solves in flight on a 2x2x1 lattice (four local blocks, halo copies
    between sweeps): per-block chunked uploads, bitwise equal to the
    sequential calls."""
    g, pd, iters, steps = (40, 36, 12), (2, 2, 1), 3, 4

    def make():
        s = sip.Solver(None, "f64", 0, lattice=(g, pd))
        As = []
        for lb, (bid, d, o) in enumerate(s.blocks):
            A = O.generate(0, 1303 + 72 + bid, d, g, o)
            As.append(A)
            s.set_system(lb, sip.StencilSystem.from_dict(A))
        s.factor(0.92)
        return s, As

    s, As = make()
    phis = [O.field(*d) for (_, d, _) in s.blocks]
    seq = []
    for k in range(steps):
        for lb, A in enumerate(As):
            s.set_source(lb, A["Q"] * (1.0 + 0.5 * k))
        n = np.asarray(s.solve(phis, iters))
        seq.append((n, [p.copy() for p in phis]))
    s.close()

    s, As = make()
    phis = [O.field(*d) for (_, d, _) in s.blocks]
    qs = [[A["Q"] * (1.0 + 0.5 * k) for A in As] for k in range(steps)]
    norms = [np.zeros(iters) for _ in range(steps)]

    def enqueue(k):
        for lb in range(len(As)):
            s.set_source_async(lb, qs[k][lb])
        s.solve_async(phis, iters, norms[k])

    enqueue(0)
    for k in range(steps):
        if k + 1 < steps:
            enqueue(k + 1)
        s.wait_async()
        assert np.array_equal(norms[k], seq[k][0]), k
    for b in range(len(phis)):
        assert np.array_equal(phis[b], seq[-1][1][b]), b
    s.synchronize()
    s.close()


def test_stream_switch_keeps_order(gpu):
    """sip_iterate enqueues without a host sync; switching to a caller stream
    in the middle of a solve keeps the earlier sweeps ordered before the
    later ones (bitwise equal to one uninterrupted solve)."""
    import torch
    dims, iters = (48, 40, 30), 6
    A = O.generate(0, 1303 + 73, dims)

    def run(switch):
        s = sip.Solver(dims, "f64")
        s.set_system(0, sip.StencilSystem.from_dict(A))
        s.factor(0.92)
        phi = O.field(*dims)
        s.load_phi([phi])
        s.iterate(iters // 2)
        st = torch.cuda.Stream()
        if switch:
            s.set_stream(st.cuda_stream)
        s.iterate(iters - iters // 2)
        s.synchronize()
        n = s.read_norms(0, iters)
        s.store_phi([phi])
        s.close()
        return np.asarray(n), phi

    n0, p0 = run(False)
    n1, p1 = run(True)
    assert np.array_equal(n0, n1)
    assert np.array_equal(p0, p1)
