"""B200-native SIP hot path of arXiv 1303.4538 (FASTEST-3D).

The product is the C-ABI library libsip_b200.so (include/sip_c.h) with its
sm_100a kernels; this package is its Python mirror of the reference's sip
module plus host-side planning helpers.
"""
from __future__ import annotations

import ctypes

import numpy as np

from .sip import (  # noqa: F401
    ARRAYS, BC, EXPORTS, LIB_PATH, ConfigError, Error, Flow, FormatError, MisuseError,
    NonConvergenceError, ProtocolError, SingularFactorError, SipConfig, SipFactors, Solver,
    SolveReport, StaleFactorsError, StencilSystem, assemble_poisson, factorization_count, field,
    ftt1_read, ftt1_validate, ftt1_write, lib, pressure_correct, residual_general,
    residual_symmetric, sip_factor, sip_sweep, solve, version,
)


def generate_host(kind: int, seed: int, dims, gdims=None, origin=(0, 0, 0)) -> dict:
    """Seeded synthetic system of one block on the host (library generator,
    DESIGN.md "Synthetic inputs"); Field3 arrays keyed by ARRAYS."""
    nx, ny, nz = dims
    g = gdims if gdims is not None else dims
    out = {n: field(nx, ny, nz) for n in ARRAYS}
    dp = ctypes.POINTER(ctypes.c_double)
    st = lib().sip_generate_host(kind, ctypes.c_uint64(seed), (ctypes.c_int * 3)(*g),
                                 (ctypes.c_int * 3)(*origin), nx, ny, nz,
                                 *[out[n].ctypes.data_as(dp) for n in ARRAYS])
    if st != 0:
        raise ConfigError(f"sip_generate_host failed ({st})")
    return out


def plan_block_ranks(p, nranks: int):
    px, py, pz = p
    out = (ctypes.c_int * (px * py * pz))()
    st = lib().sip_plan_block_ranks(px, py, pz, nranks, out)
    if st != 0:
        raise ConfigError(f"cannot place {px*py*pz} blocks on {nranks} ranks")
    return list(out)


def plan_halo(g, p, block_rank, rank: int, periodic_mask: int = 0):
    """Face-halo entries of one rank: rows of (dir, kind, face, peer, owner,
    neighbor, ilo, ihi, jlo, jhi, klo, khi) as in the reference's FTT1 entry;
    bit a of periodic_mask wraps axis a (transfers.cpp:15-25)."""
    n = ctypes.c_int(0)
    br = None if block_rank is None else (ctypes.c_int * len(block_rank))(*block_rank)
    st = lib().sip_plan_halo_periodic(*g, *p, br, rank, periodic_mask, ctypes.byref(n), None)
    if st != 0:
        raise ConfigError("sip_plan_halo failed")
    buf = (ctypes.c_int * (12 * max(n.value, 1)))()
    st = lib().sip_plan_halo_periodic(*g, *p, br, rank, periodic_mask, ctypes.byref(n), buf)
    if st != 0:
        raise ConfigError("sip_plan_halo failed")
    return np.array(buf[: 12 * n.value], dtype=np.int64).reshape(n.value, 12)


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    st = lib().sip_nccl_unique_id(buf)
    if st != 0:
        raise Error("ncclGetUniqueId failed")
    return buf.raw
