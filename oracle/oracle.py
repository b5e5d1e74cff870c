"""ctypes front-end of the CPU SIP oracle (oracle/sip_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference legs of bench.py.  The product path
(paper_1303_4538_b200) never imports this module.

Arrays are numpy float64 in the reference's Field3 layout
(proj/include/bsfv/field.hpp:25-44): shape (nz+2, ny+2, nx+2), i fastest,
interior 1..n, one ghost layer.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "_ref", "libsip_oracle.so")
_lib = None

ARRAYS = ("AP", "AW", "AE", "AS", "AN", "AB", "AT", "Q")
FACTORS = ("LB", "LW", "LS", "LP", "UN", "UE", "UT")

_dp = ctypes.POINTER(ctypes.c_double)
_fp = ctypes.POINTER(ctypes.c_float)


def build() -> str:
    """Compile the oracle shared library (gcc, -ffp-contract=off)."""
    subprocess.run(["make", "-s", "-C", _HERE, "_ref/libsip_oracle.so"], check=True)
    return _SO


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(
            os.path.join(_HERE, "sip_oracle.c")
        ):
            build()
        L = ctypes.CDLL(_SO)
        L.orc_u01.restype = ctypes.c_double
        L.orc_u01.argtypes = [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint64]
        L.orc_generate.restype = None
        L.orc_factor.restype = ctypes.c_int
        L.orc_sweep_d.restype = ctypes.c_double
        L.orc_sweep_f.restype = ctypes.c_double
        L.orc_sweep_pipe_d.restype = ctypes.c_double
        L.orc_sweep_pipe_f.restype = ctypes.c_double
        L.orc_solve.restype = ctypes.c_int
        L.orc_solve_multi.restype = ctypes.c_int
        L.orc_solve_multi_gen.restype = ctypes.c_int
        _lib = L
    return _lib


def _p(a: np.ndarray):
    assert a.flags.c_contiguous
    if a.dtype == np.float64:
        return a.ctypes.data_as(_dp)
    if a.dtype == np.float32:
        return a.ctypes.data_as(_fp)
    raise TypeError(a.dtype)


def field(nx: int, ny: int, nz: int, dtype=np.float64) -> np.ndarray:
    return np.zeros((nz + 2, ny + 2, nx + 2), dtype=dtype)


def generate(kind: int, seed: int, dims, gdims=None, origin=(0, 0, 0)) -> dict:
    """Seeded synthetic system of one block."""
    nx, ny, nz = dims
    g = gdims if gdims is not None else dims
    A = {n: field(nx, ny, nz) for n in ARRAYS}
    gi = (ctypes.c_int * 3)(*g)
    oi = (ctypes.c_int * 3)(*origin)
    lib().orc_generate(ctypes.c_int(kind), ctypes.c_uint64(seed), gi, oi, nx, ny, nz,
                       *[_p(A[n]) for n in ARRAYS])
    return A


def factor(A: dict, alpha: float):
    """Stone factors or raises ValueError naming the singular cell."""
    nz, ny, nx = (s - 2 for s in A["AP"].shape)
    F = {n: field(nx, ny, nz) for n in FACTORS}
    bad = ctypes.c_longlong(-1)
    rc = lib().orc_factor(nx, ny, nz, ctypes.c_double(alpha), *[_p(A[n]) for n in ARRAYS[:7]],
                          *[_p(F[n]) for n in FACTORS], ctypes.byref(bad))
    if rc:
        raise ValueError(f"singular factorization at Field3 index {bad.value}")
    return F


def residual(A: dict, phi: np.ndarray) -> np.ndarray:
    nz, ny, nx = (s - 2 for s in A["AP"].shape)
    res = field(nx, ny, nz)
    lib().orc_residual(nx, ny, nz, *[_p(A[n]) for n in ARRAYS], _p(phi), _p(res))
    return res


def residual_symmetric(A: dict, phi: np.ndarray) -> np.ndarray:
    nz, ny, nx = (s - 2 for s in A["AP"].shape)
    res = field(nx, ny, nz)
    lib().orc_residual_symmetric(nx, ny, nz, _p(A["AP"]), _p(A["AE"]), _p(A["AN"]), _p(A["AT"]),
                                 _p(A["Q"]), _p(phi), _p(res))
    return res


def sweep(A: dict, F: dict, phi: np.ndarray) -> float:
    """One fp64 SIP iteration in place on phi; returns the L1 residual norm."""
    nz, ny, nx = (s - 2 for s in A["AP"].shape)
    work = field(nx, ny, nz, phi.dtype)
    if phi.dtype == np.float64:
        fn = lib().orc_sweep_d
    else:
        fn = lib().orc_sweep_f
    return fn(nx, ny, nz, *[_p(A[n]) for n in ARRAYS], *[_p(F[n]) for n in FACTORS], _p(phi),
              _p(work))


def sweep_pipe(A: dict, F: dict, phi: np.ndarray, nthreads: int, work=None) -> float:
    """sweep() on `nthreads` host threads (j-slab pipeline, bitwise-equal phi);
    `work` (zero ghost layer, phi's dtype) may be reused across calls."""
    nz, ny, nx = (s - 2 for s in A["AP"].shape)
    if work is None:
        work = field(nx, ny, nz, phi.dtype)
    fn = lib().orc_sweep_pipe_d if phi.dtype == np.float64 else lib().orc_sweep_pipe_f
    return fn(nx, ny, nz, *[_p(A[n]) for n in ARRAYS], *[_p(F[n]) for n in FACTORS], _p(phi),
              _p(work), int(nthreads))


def forward(A: dict, F: dict, phi: np.ndarray) -> np.ndarray:
    """Residual + forward substitution only: returns R (fp64)."""
    nz, ny, nx = (s - 2 for s in A["AP"].shape)
    work = field(nx, ny, nz)
    lib().orc_forward_d.restype = ctypes.c_double
    lib().orc_forward_d(nx, ny, nz, *[_p(A[n]) for n in ARRAYS], *[_p(F[n]) for n in FACTORS[:4]],
                        _p(phi), _p(work))
    return work


def solve(A: dict, phi: np.ndarray, alpha: float, iters: int, precision: str = "f64"):
    """Factor + `iters` SIP iterations; phi updated in place.  Returns norms."""
    nz, ny, nx = (s - 2 for s in A["AP"].shape)
    norms = np.zeros(max(iters, 1))
    arr = (_dp * 8)(*[_p(A[n]) for n in ARRAYS])
    bad = ctypes.c_longlong(-1)
    rc = lib().orc_solve(nx, ny, nz, 0 if precision == "f64" else 1, ctypes.c_double(alpha),
                         iters, arr, _p(phi), _p(norms), ctypes.byref(bad))
    if rc == 1:
        raise ValueError(f"singular factorization at Field3 index {bad.value}")
    if rc:
        raise MemoryError("oracle allocation failed")
    return norms[:iters]


def solve_multi(blocks, nbr, alpha: float, iters: int, precision: str = "f64", nthreads: int = 1):
    """Block-Jacobi SIP over several blocks.

    blocks: list of (A dict, phi array); nbr: list of 6-tuples (W,E,S,N,B,T)
    neighbour block ids or -1.  Returns (norms[iters], block_norms[iters, nb]).
    """
    nb = len(blocks)
    dims = (ctypes.c_int * (3 * nb))()
    nb_ = (ctypes.c_int * (6 * nb))()
    arr = (_dp * (8 * nb))()
    phis = (_dp * nb)()
    for b, (A, phi) in enumerate(blocks):
        nz, ny, nx = (s - 2 for s in A["AP"].shape)
        dims[3 * b:3 * b + 3] = [nx, ny, nz]
        nb_[6 * b:6 * b + 6] = list(nbr[b])
        for a, n in enumerate(ARRAYS):
            arr[8 * b + a] = _p(A[n])
        phis[b] = _p(phi)
    norms = np.zeros(max(iters, 1))
    bnorms = np.zeros((max(iters, 1), nb))
    bad = ctypes.c_longlong(-1)
    rc = lib().orc_solve_multi(nb, dims, nb_, 0 if precision == "f64" else 1,
                               ctypes.c_double(alpha), iters, arr, phis, _p(norms), _p(bnorms),
                               nthreads, ctypes.byref(bad))
    if rc == 1:
        raise ValueError(f"singular factorization at Field3 index {bad.value}")
    return norms[:iters], bnorms[:iters]


def solve_pipe(A: dict, phi: np.ndarray, alpha: float, iters: int, precision: str = "f64",
               nthreads: int = 0):
    """solve() with the sweeps pipelined over host threads (orc_sweep_pipe_*,
    bitwise equal to the serial sweep): factor in fp64, fp32 mode converts the
    system, factors and phi once at entry and the interior back at exit
    (exactly orc_solve).  For the full-size BASELINE configs."""
    nthreads = nthreads or (len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count())
    F = factor(A, alpha)
    norms = np.zeros(iters)
    if precision == "f64":
        work = np.zeros_like(phi)
        for it in range(iters):
            norms[it] = sweep_pipe(A, F, phi, nthreads, work)
        return norms
    A32 = {n: np.ascontiguousarray(v, dtype=np.float32) for n, v in A.items()}
    F32 = {n: np.ascontiguousarray(v, dtype=np.float32) for n, v in F.items()}
    ph = phi.astype(np.float32)
    work = np.zeros_like(ph)
    for it in range(iters):
        norms[it] = sweep_pipe(A32, F32, ph, nthreads, work)
    phi[1:-1, 1:-1, 1:-1] = ph[1:-1, 1:-1, 1:-1].astype(np.float64)
    return norms


def solve_multi_gen(kind: int, seed0: int, gdims, pdims, phis, alpha: float, iters: int,
                    precision: str = "f64", nthreads: int = 0):
    """Block-Jacobi SIP over the generated lattice (block b: seed0 + b), each
    block's system regenerated / refactored on the fly (orc_solve_multi_gen:
    memory-lean).  phis: one Field3 fp64 array per block (in / out).  Returns
    (norms[iters], block_norms[iters, nb])."""
    nthreads = nthreads or (len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count())
    origins, dims, nbr = lattice(gdims, pdims)
    nb = len(dims)
    org_ = (ctypes.c_int * (3 * nb))(*[x for o in origins for x in o])
    dims_ = (ctypes.c_int * (3 * nb))(*[x for d in dims for x in d])
    nbr_ = (ctypes.c_int * (6 * nb))(*[x for n in nbr for x in n])
    ph = (_dp * nb)(*[_p(p) for p in phis])
    g = (ctypes.c_int * 3)(*gdims)
    norms = np.zeros(max(iters, 1))
    bnorms = np.zeros((max(iters, 1), nb))
    bad = ctypes.c_longlong(-1)
    rc = lib().orc_solve_multi_gen(kind, ctypes.c_uint64(seed0), g, nb, org_, dims_, nbr_,
                                   0 if precision == "f64" else 1, ctypes.c_double(alpha), iters, ph,
                                   _p(norms), _p(bnorms), int(nthreads), ctypes.byref(bad))
    if rc == 1:
        raise ValueError(f"singular factorization at Field3 index {bad.value}")
    return norms[:iters], bnorms[:iters]


def lattice(gdims, pdims):
    """Block lattice like bsfv::decompose (proj/src/grid.cpp:50-89): even split,
    remainder to the LAST block per axis.  Returns (origins, dims, nbr) with
    block id = bx + px*(by + py*bz) and non-periodic face neighbours."""
    origins, dims, nbr = [], [], []
    px, py, pz = pdims

    def split(n, p):
        base = n // p
        ext = [base] * p
        ext[-1] += n - base * p
        off = [sum(ext[:q]) for q in range(p)]
        return off, ext

    ox, ex = split(gdims[0], px)
    oy, ey = split(gdims[1], py)
    oz, ez = split(gdims[2], pz)
    for bz in range(pz):
        for by in range(py):
            for bx in range(px):
                origins.append((ox[bx], oy[by], oz[bz]))
                dims.append((ex[bx], ey[by], ez[bz]))
                bid = lambda x, y, z: x + px * (y + py * z)
                nbr.append((
                    bid(bx - 1, by, bz) if bx > 0 else -1,
                    bid(bx + 1, by, bz) if bx < px - 1 else -1,
                    bid(bx, by - 1, bz) if by > 0 else -1,
                    bid(bx, by + 1, bz) if by < py - 1 else -1,
                    bid(bx, by, bz - 1) if bz > 0 else -1,
                    bid(bx, by, bz + 1) if bz < pz - 1 else -1,
                ))
    return origins, dims, nbr
