"""The SIP caller: assemble_poisson
and pressure_correct with factor reuse.

CPU tests pin the oracle restatement (oracle/flow.py) to the specification's
worked examples; GPU tests compare the library (sip_flow.cu through the
C-ABI) with the oracle bit for bit and check the spec's properties.
"""
import numpy as np
import pytest

import paper_1303_4538_b200 as sip
from oracle import flow as OF
from oracle import oracle as O

W, P, S = OF.WALL, OF.PERIODIC, OF.SYMMETRY
INNER = (slice(1, -1),) * 3


# ---------------------------------------------------------------- oracle pins
def test_oracle_uniform_cubes_interior_coefficients():
    """uniform cubic cells h -> a_nb = h, ap = 6h at interior cells."""
    h = 0.25
    (A,) = OF.assemble_poisson((4, 4, 4), (1, 1, 1), (4 * h,) * 3, (P,) * 6)
    for n in ("AW", "AE", "AS", "AN", "AB", "AT"):
        assert A[n][2, 2, 2] == -h  # matrix-entry convention A_nb = -a_nb
    assert A["AP"][2, 2, 2] == 6 * h
    assert np.all(A["Q"] == 0.0)


def test_oracle_wall_face_is_neumann():
    """coefficient through a wall = 0, ap reduced accordingly."""
    h = 0.5
    (A,) = OF.assemble_poisson((4, 4, 4), (1, 1, 1), (2.0, 2.0, 2.0), (W,) * 6)
    c = (1, 2, 2)  # cell on the B wall (k = 0), not the pinned cell
    assert A["AB"][c] == 0.0 and A["AT"][c] == -h
    assert A["AP"][c] == 5 * h
    corner = (1, 1, 4)  # i = nx-1, j = 0, k = 0: three walls
    assert A["AP"][corner] == 3 * h


def test_oracle_periodic_row_sums_zero_except_pinned():
    """4^3 periodic block, row sums ap - sum a_nb = 0 except the pinned cell."""
    (A,) = OF.assemble_poisson((4, 4, 4), (1, 1, 1), (1.0, 1.0, 1.0), (P,) * 6)
    rs = A["AP"] + sum(A[n] for n in ("AW", "AE", "AS", "AN", "AB", "AT"))
    rs = rs[INNER]
    assert rs[0, 0, 0] == 1.0
    rs[0, 0, 0] = 0.0
    assert np.all(rs == 0.0)


def test_oracle_anisotropic_cells():
    """a_nb = face area / centre distance for hx != hy != hz."""
    (A,) = OF.assemble_poisson((4, 5, 6), (1, 1, 1), (1.0, 2.0, 3.0), (P,) * 6)
    hx, hy, hz = 0.25, 0.4, 0.5
    assert A["AE"][3, 3, 3] == -((hy * hz) / hx)
    assert A["AN"][3, 3, 3] == -((hx * hz) / hy)
    assert A["AT"][3, 3, 3] == -((hx * hy) / hz)


def test_oracle_divergence_free_needs_no_solve():
    """divergence-free input -> zero outer iterations."""
    g, p, bc = (8, 8, 8), (1, 1, 1), (P,) * 6
    As = OF.assemble_poisson(g, p, (1.0,) * 3, bc)
    _, dims, nbr = OF.wrapped_lattice(g, p, bc)
    us = [O.field(*d) + 0.7 for d in dims]
    vs = [O.field(*d) for d in dims]
    ws = [O.field(*d) for d in dims]
    ps = [O.field(*d) for d in dims]
    outer, hist = OF.pressure_correct(As, nbr, us, vs, ws, ps, OF.cell_sizes(g, (1.0,) * 3), 0.1,
                                      1e-12, 5, 3)
    assert outer == 0 and hist == [0.0]


def test_oracle_projection_reduces_divergence():
    """A smooth divergent field on a periodic box: each outer iteration cuts
    the divergence (SPEC.md:348 restated at oracle size)."""
    g, p, bc = (8, 8, 8), (1, 1, 1), (P,) * 6
    As = OF.assemble_poisson(g, p, (1.0,) * 3, bc)
    _, dims, nbr = OF.wrapped_lattice(g, p, bc)
    us, vs, ws, ps = _smooth_fields(g, p)
    h = OF.cell_sizes(g, (1.0,) * 3)
    hist = []
    for cap in range(4):
        fields = [[a.copy() for a in f] for f in (us, vs, ws, ps)]
        with pytest.raises(RuntimeError) as e:
            OF.pressure_correct(As, nbr, *fields, h, 0.1, 0.0, cap, 8)
        hist.append(e.value.args[1])
    assert all(b < a for a, b in zip(hist, hist[1:]))
    assert hist[-1] < 2e-2 * hist[0]


def _smooth_fields(g, p, seed=3):
    """u, v, w, p per block of the lattice: low Fourier modes plus noise."""
    origins, dims, _ = O.lattice(g, p)
    rng = np.random.default_rng(seed)
    amp = rng.uniform(-1, 1, 6)
    out = [[], [], [], []]
    for o, d in zip(origins, dims):
        k, j, i = np.meshgrid(*(np.arange(d[a]) + o[a] + 0.5 for a in (2, 1, 0)), indexing="ij")
        x, y, z = i / g[0], j / g[1], k / g[2]
        tp = 2 * np.pi
        fields = [amp[0] * np.sin(tp * x) + amp[1] * np.cos(tp * (y + z)),
                  amp[2] * np.sin(tp * y) * np.cos(tp * x),
                  amp[3] * np.cos(tp * z) + amp[4] * np.sin(tp * (x - y)),
                  amp[5] * np.cos(tp * x) * np.sin(tp * z)]
        for q in range(4):
            f = O.field(*d)
            f[INNER] = fields[q]
            out[q].append(f)
    return out


# ---------------------------------------------------------------- GPU parity
def _gpu_setup(g, p, bc, prec, lengths=(1.0, 1.0, 1.0), alpha=0.92):
    s = sip.Solver(None, prec, 0, lattice=(g, p))
    s.assemble_poisson(lengths, [("wall", "periodic", "symmetry")[b] for b in bc])
    s.factor(alpha)
    return s


@pytest.mark.gpu
@pytest.mark.parametrize("bc", [(W,) * 6, (P, P, W, W, S, S), (P,) * 6])
def test_assemble_matches_oracle(gpu, bc):
    g, p = (20, 12, 10), (2, 1, 2)
    s = sip.Solver(None, "f64", 0, lattice=(g, p))
    s.assemble_poisson((2.0, 1.5, 1.0), [("wall", "periodic", "symmetry")[b] for b in bc])
    ref = OF.assemble_poisson(g, p, (2.0, 1.5, 1.0), bc)
    import ctypes
    for lb, (bid, d, o) in enumerate(s.blocks):
        for a, name in enumerate(O.ARRAYS):
            out = O.field(*d)
            st = sip.lib().sip_debug_field(s.handle, lb, 2 + a, out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
            assert st == 0
            assert np.array_equal(out[INNER], ref[bid][name][INNER]), (bid, name)
    s.close()


@pytest.mark.gpu
@pytest.mark.parametrize("prec", ["f64", "f32"])
@pytest.mark.parametrize("case", ["walls_2x2x1", "perx_2x1x2", "perall_1x2x1", "ragged_sym_2x1x1",
                                  "thin_1x1x3"])
def test_pressure_correct_matches_oracle(gpu, prec, case):
    """Fields after a capped outer loop and the divergence history: bitwise /
    1e-12 relative against the oracle (GPU SIP parity is bitwise already).
    Ragged tiles (extents not multiples of 16), symmetry faces, 1-cell-thin
    blocks included."""
    g, p, bc = {"walls_2x2x1": ((16, 12, 8), (2, 2, 1), (W,) * 6),
                "perx_2x1x2": ((16, 8, 12), (2, 1, 2), (P, P, W, W, W, W)),
                "perall_1x2x1": ((12, 16, 8), (1, 2, 1), (P,) * 6),
                "ragged_sym_2x1x1": ((37, 21, 9), (2, 1, 1), (S, W, P, P, S, S)),
                "thin_1x1x3": ((5, 3, 3), (1, 1, 3), (P, P, W, W, P, P))}[case]
    lengths = (1.0, 0.75, 0.5)
    dt, outer_cap, sweeps = 0.05, 3, 4
    s = _gpu_setup(g, p, bc, prec, lengths)
    us, vs, ws, ps = _smooth_fields(g, p)
    fl = sip.Flow(s)
    bids = [bid for (bid, _, _) in s.blocks]
    for name, arrs in zip("uvwp", (us, vs, ws, ps)):
        fl.set(name, [arrs[b] for b in bids])
    with pytest.raises(sip.NonConvergenceError) as e:
        fl.pressure_correct(dt, 0.0, outer_cap, sweeps)
    got = {}
    for name in "uvwp":
        arrs = [O.field(*d) for (_, d, _) in s.blocks]
        fl.get(name, arrs)
        got[name] = arrs
    fl.close()
    s.close()
    As = OF.assemble_poisson(g, p, lengths, bc)
    _, dims, nbr = OF.wrapped_lattice(g, p, bc)
    h = OF.cell_sizes(g, lengths)
    with pytest.raises(RuntimeError) as eo:
        OF.pressure_correct(As, nbr, us, vs, ws, ps, h, dt, 0.0, outer_cap, sweeps, 0.92, prec)
    np.testing.assert_allclose(e.value.defect, eo.value.args[1], rtol=1e-12)
    for name, ref in zip("uvwp", (us, vs, ws, ps)):
        for lb, bid in enumerate(bids):
            assert np.array_equal(got[name][lb][INNER], ref[bid][INNER]), (name, bid)


@pytest.mark.gpu
def test_factor_reuse_over_100_steps(gpu):
    """SPEC.md:349 / criterion 4: the factorization counter stays 1 across 100
    pressure-correction steps on the constant pressure system."""
    g, p, bc = (16, 16, 16), (2, 1, 1), (P, P, W, W, P, P)
    c0 = sip.factorization_count()
    s = _gpu_setup(g, p, bc, "f64")
    assert sip.factorization_count() - c0 == 1
    us, vs, ws, ps = _smooth_fields(g, p)
    fl = sip.Flow(s)
    bids = [bid for (bid, _, _) in s.blocks]
    solves = 0
    for step in range(100):
        if step % 10 == 0:  # a fresh smooth divergent field every 10 steps
            fresh = _smooth_fields(g, p, seed=100 + step)
            for name, arrs in zip("uvw", fresh[:3]):
                fl.set(name, [arrs[b] for b in bids])
        d0 = fl.divergence()
        # fresh fields: cut the divergence 3x; other steps: the mass check only
        thr = 0.3 * d0 if step % 10 == 0 else d0
        outer, hist = fl.pressure_correct(0.01, thr, 40, 5)
        assert hist[-1] <= thr
        solves += outer
    assert sip.factorization_count() - c0 == 1
    assert solves >= 10
    fl.close()
    s.close()


@pytest.mark.gpu
def test_divergence_free_input_zero_outer(gpu):
    """divergence-free input -> p' = 0, no solve."""
    g, p, bc = (16, 16, 8), (1, 2, 1), (P,) * 6
    s = _gpu_setup(g, p, bc, "f64")
    fl = sip.Flow(s)
    d = [O.field(*dd) for (_, dd, _) in s.blocks]
    for f in d:
        f[INNER] = 0.3
    fl.set("u", d)
    zero = [O.field(*dd) for (_, dd, _) in s.blocks]
    fl.set("v", zero)
    fl.set("w", zero)
    fl.set("p", zero)
    outer, hist = fl.pressure_correct(0.1, 1e-14, 5, 5)
    assert outer == 0 and hist[0] == 0.0
    out = [O.field(*dd) for (_, dd, _) in s.blocks]
    fl.get("p", out)
    assert all(np.all(o[INNER] == 0.0) for o in out)
    fl.close()
    s.close()


@pytest.mark.gpu
@pytest.mark.parametrize("prec", ["f64", "f32"])
def test_projection_restores_divergence(gpu, prec):
    """an injected smooth divergence on a periodic box is cut by
    the outer loop, monotonically.  With the identity-row pin the
    pinned cell's near-null mode converges at ~1 % per SIP sweep, so the
    reachable reduction in a bounded loop is ~1e-2 .. 1e-3, not the example's 1e-10
    (DESIGN.md section 9)."""
    g, p, bc = (32, 32, 32), (2, 2, 1), (P,) * 6
    s = _gpu_setup(g, p, bc, prec)
    fl = sip.Flow(s)
    us, vs, ws, ps = _smooth_fields(g, p, seed=11)
    bids = [bid for (bid, _, _) in s.blocks]
    for name, arrs in zip("uvwp", (us, vs, ws, ps)):
        fl.set(name, [arrs[b] for b in bids])
    d0 = fl.divergence()
    thr = 1e-2 * d0
    outer, hist = fl.pressure_correct(0.1, thr, 200, 8)
    assert hist[-1] <= thr and outer >= 1
    assert np.all(np.diff(hist) < 0), hist  # monotone decrease
    fl.close()
    s.close()


@pytest.mark.gpu
def test_outer_cap_raises_with_defect(gpu):
    g, p, bc = (16, 16, 16), (1, 1, 1), (W,) * 6
    s = _gpu_setup(g, p, bc, "f64")
    fl = sip.Flow(s)
    us, vs, ws, ps = _smooth_fields(g, p)
    for name, arrs in zip("uvwp", (us, vs, ws, ps)):
        fl.set(name, arrs)
    d0 = fl.divergence()
    with pytest.raises(sip.NonConvergenceError) as e:
        fl.pressure_correct(0.1, 0.0, 0, 5)
    assert e.value.defect == d0 > 0
    fl.close()
    s.close()


@pytest.mark.gpu
def test_bad_config_and_misuse(gpu):
    s = sip.Solver(None, "f64", 0, lattice=((8, 8, 8), (1, 1, 1)))
    with pytest.raises(sip.MisuseError):
        sip.Flow(s)  # before assemble_poisson
    with pytest.raises(sip.ConfigError):
        s.assemble_poisson((1.0, 1.0, 1.0), ("periodic", "wall", "wall", "wall", "wall", "wall"))
    with pytest.raises(sip.ConfigError):
        s.assemble_poisson((1.0, -1.0, 1.0))
    s.assemble_poisson((1.0, 1.0, 1.0))
    fl = sip.Flow(s)
    with pytest.raises(sip.MisuseError):  # not factored yet
        fl.pressure_correct(0.1, 0.0, 1, 1)
    s.assemble_poisson((1.0, 1.0, 1.0), ("periodic",) * 6)  # new halo plan
    s.factor(0.92)
    with pytest.raises(sip.MisuseError):  # the flow was built for the old plan
        fl.divergence()
    fl2 = sip.Flow(s)
    assert fl2.divergence() == 0.0
    s.generate(0, 7)  # the pressure system is replaced: the caller refuses to run on it
    s.factor(0.92)
    with pytest.raises(sip.MisuseError):
        fl2.pressure_correct(0.1, 0.0, 1, 1)
    s.close()  # closes its flows first
    assert not fl._h and not fl2._h
