"""CPU restatement of the SIP caller: assemble_poisson and
pressure_correct on a block lattice.

TEST INFRASTRUCTURE ONLY: imported by tests/ (and nothing in the product).
The reference defines both operations only in its specification (the
artifact ships no implementation), so this module restates the spec with the
design decisions it leaves open written down:

  * coefficients a_nb = face area / centre distance, zero through a wall or
    symmetry face, coupled across periodic faces; stored as A_nb = -a_nb,
    AP = ((((aW + aE) + aS) + aN) + aB) + aT;
  * global cell (0,0,0) pinned as an identity row, Q = 0;
  * co-located central differences: div = ((uE-uW)/2hx +
    (vN-vS)/2hy) + (wT-wB)/2hz, Q = -(V*div)/dt, u -= dt*((p'E-p'W)/2hx), p += p';
  * ghosts: neighbour planes through the (wrapped) block lattice; at walls the
    normal velocity ghost is -interior (zero face velocity) and the p' ghost
    is the interior value (homogeneous Neumann);
  * divergence L1 = sum |div| * V, blocks summed in block-id order.

Every elementwise formula is written in the same operation order as the
CUDA kernels (paper_1303_4538_b200/csrc/sip_flow.cu), so fields agree bit for
bit; the SIP solve is oracle.solve_multi (block-Jacobi SIP, sip_oracle.c).
"""
from __future__ import annotations

import numpy as np

from . import oracle as O

WALL, PERIODIC, SYMMETRY = 0, 1, 2
# Field3 arrays are (k, j, i); faces W,E,S,N,B,T -> (axis of the array, low side?)
_FACE_AX = ((2, True), (2, False), (1, True), (1, False), (0, True), (0, False))


def wrapped_lattice(g, p, bc):
    """oracle.lattice with the neighbour table wrapped on periodic axes
    (transfers.cpp:15-25)."""
    origins, dims, nbr = O.lattice(g, p)
    px, py, pz = p
    out = []
    for b in range(len(dims)):
        c = [b % px, (b // px) % py, b // (px * py)]
        n = list(nbr[b])
        for a in range(3):
            if bc[2 * a] == PERIODIC:
                lo, hi = list(c), list(c)
                lo[a] = (lo[a] - 1) % p[a]
                hi[a] = (hi[a] + 1) % p[a]
                n[2 * a] = lo[0] + px * (lo[1] + py * lo[2])
                n[2 * a + 1] = hi[0] + px * (hi[1] + py * hi[2])
        out.append(tuple(n))
    return origins, dims, out


def cell_sizes(g, lengths):
    return [lengths[a] / g[a] for a in range(3)]


def assemble_poisson(g, p, lengths, bc):
    """Per-block StencilSystem dicts (Field3 arrays) of the pressure equation."""
    origins, dims, nbr = O.lattice(g, p)
    hx, hy, hz = cell_sizes(g, lengths)
    ax, ay, az = (hy * hz) / hx, (hx * hz) / hy, (hx * hy) / hz
    blocks = []
    for b, (nx, ny, nz) in enumerate(dims):
        cpl = [nbr[b][f] >= 0 or bc[f] == PERIODIC for f in range(6)]
        k, j, i = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
        w = np.where((i > 0) | cpl[0], ax, 0.0)
        e = np.where((i < nx - 1) | cpl[1], ax, 0.0)
        s = np.where((j > 0) | cpl[2], ay, 0.0)
        n = np.where((j < ny - 1) | cpl[3], ay, 0.0)
        bb = np.where((k > 0) | cpl[4], az, 0.0)
        t = np.where((k < nz - 1) | cpl[5], az, 0.0)
        A = {name: O.field(nx, ny, nz) for name in O.ARRAYS}
        inner = (slice(1, -1),) * 3
        A["AP"][inner] = ((((w + e) + s) + n) + bb) + t
        A["AW"][inner] = -w
        A["AE"][inner] = -e
        A["AS"][inner] = -s
        A["AN"][inner] = -n
        A["AB"][inner] = -bb
        A["AT"][inner] = -t
        if b == 0:  # global cell (0,0,0): identity row
            for name in O.ARRAYS:
                A[name][1, 1, 1] = 0.0
            A["AP"][1, 1, 1] = 1.0
        blocks.append(A)
    return blocks


def _plane(a, face, ghost):
    """Index tuple of a Field3 face plane (interior layer or ghost layer)."""
    ax, low = _FACE_AX[face]
    sl = [slice(1, -1)] * 3
    if low:
        sl[ax] = 0 if ghost else 1
    else:
        sl[ax] = -1 if ghost else -2
    return tuple(sl)


def fill_ghosts(fields, nbr, wall_sign):
    """Face ghosts of per-block Field3 arrays: the neighbour's facing interior
    plane, or sign * own interior plane at a wall (sign per face)."""
    for b, f in enumerate(fields):
        for face in range(6):
            nb = nbr[b][face]
            if nb >= 0:
                f[_plane(None, face, True)] = fields[nb][_plane(None, face ^ 1, False)]
            else:
                v = f[_plane(None, face, False)]
                f[_plane(None, face, True)] = -v if wall_sign[face] < 0 else v
    return fields


def divergence(u, v, w, h, dt=None, pin=True):
    """(div interior array, Q interior array or None) of one block."""
    c2x, c2y, c2z = 2.0 * h[0], 2.0 * h[1], 2.0 * h[2]
    I = slice(1, -1)
    dv = (((u[I, I, 2:] - u[I, I, :-2]) / c2x + (v[I, 2:, I] - v[I, :-2, I]) / c2y)
          + (w[2:, I, I] - w[:-2, I, I]) / c2z)
    q = None
    if dt is not None:
        vol = (h[0] * h[1]) * h[2]
        q = -(vol * dv) / dt
    return dv, q


def divergence_l1(us, vs, ws, h):
    """L1 of the divergence with the ghosts as they are (callers fill them)."""
    vol = (h[0] * h[1]) * h[2]
    tot = 0.0
    for u, v, w in zip(us, vs, ws):
        dv, _ = divergence(u, v, w, h)
        tot += float(np.sum(np.abs(dv) * vol))
    return tot


U_SIGN = (-1, -1, 1, 1, 1, 1)
V_SIGN = (1, 1, -1, -1, 1, 1)
W_SIGN = (1, 1, 1, 1, -1, -1)
P_SIGN = (1, 1, 1, 1, 1, 1)


def pressure_correct(As, nbr, us, vs, ws, ps, h, dt, threshold, max_outer, sweeps,
                     alpha=0.92, precision="f64"):
    """Outer loop of SPEC.md:341-349 on lists of per-block Field3 arrays
    (updated in place).  Returns (outer iterations, divergence history) or
    raises RuntimeError('noconv', defect) at the cap."""
    hist = []
    vol = (h[0] * h[1]) * h[2]
    I = slice(1, -1)
    for outer in range(max_outer + 1):
        fill_ghosts(us, nbr, U_SIGN)
        fill_ghosts(vs, nbr, V_SIGN)
        fill_ghosts(ws, nbr, W_SIGN)
        tot = 0.0
        qs = []
        for b in range(len(As)):
            dv, q = divergence(us[b], vs[b], ws[b], h, dt)
            if b == 0:
                q[0, 0, 0] = 0.0
            qs.append(q)
            tot += float(np.sum(np.abs(dv) * vol))
        hist.append(tot)
        if tot <= threshold:
            return outer, hist
        if outer == max_outer:
            raise RuntimeError("noconv", tot)
        blocks = []
        for b, A in enumerate(As):
            A["Q"][I, I, I] = qs[b]
            blocks.append((A, np.zeros_like(A["AP"])))
        O.solve_multi(blocks, nbr, alpha, sweeps, precision)
        pp = fill_ghosts([phi for _, phi in blocks], nbr, P_SIGN)
        c2x, c2y, c2z = 2.0 * h[0], 2.0 * h[1], 2.0 * h[2]
        for b in range(len(As)):
            q = pp[b]
            us[b][I, I, I] = us[b][I, I, I] - dt * ((q[I, I, 2:] - q[I, I, :-2]) / c2x)
            vs[b][I, I, I] = vs[b][I, I, I] - dt * ((q[I, 2:, I] - q[I, :-2, I]) / c2y)
            ws[b][I, I, I] = ws[b][I, I, I] - dt * ((q[2:, I, I] - q[:-2, I, I]) / c2z)
            ps[b][I, I, I] = ps[b][I, I, I] + q[I, I, I]
    raise AssertionError("unreachable")
