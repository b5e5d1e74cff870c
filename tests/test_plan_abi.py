"""CPU tests of the C-ABI library: exported symbols, host-side planning
(block lattice, compact block->rank placement, face-halo plan) against the
reference's own decompose / build_transfer_tables output (golden fixtures
generated from the reference sources by oracle/make_golden.py)."""
import ctypes
import json
import os
import re

import numpy as np
import pytest

import paper_1303_4538_b200 as sip

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")


def header_functions():
    txt = open(os.path.join(ROOT, "include", "sip_c.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(sip_[a-z_0-9]+)\s*\(", txt)))


def test_library_exports_every_header_symbol():
    L = sip.lib()
    names = header_functions()
    assert len(names) >= 30
    for n in names:
        assert hasattr(L, n), f"{n} declared in include/sip_c.h but not exported"
    assert set(sip.EXPORTS) <= set(names)


def test_version_and_status_strings():
    assert "sm_100a" in sip.version()
    L = sip.lib()
    for st in range(0, 8):
        assert L.sip_status_string(st)
    assert L.sip_status_string(1) == b"singular factorization"
    assert L.sip_status_string(10) == b"pressure correction did not converge"


def test_create_without_device_fails_cleanly():
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except Exception:
        pass
    ctx = ctypes.c_void_p()
    st = sip.lib().sip_create(0, 8, 8, 8, 0, ctypes.byref(ctx))
    assert st == sip.sip.SIP_ERR_CUDA and not ctx.value
    assert sip.lib().sip_last_error(None)


def test_create_rejects_bad_config():
    ctx = ctypes.c_void_p()
    L = sip.lib()
    assert L.sip_create(0, 8, 8, 8, 7, ctypes.byref(ctx)) == sip.sip.SIP_ERR_CONFIG
    assert L.sip_create_lattice(0, 4, 4, 4, 5, 1, 1, None, 0, 1, None, 0,
                                ctypes.byref(ctx)) == sip.sip.SIP_ERR_CONFIG
    assert b"more blocks" in L.sip_last_error(None)
    # device kernels index a block's cells with 32-bit arithmetic
    assert L.sip_create_lattice(0, 4096, 4096, 512, 1, 1, 1, None, 0, 1, None, 0,
                                ctypes.byref(ctx)) == sip.sip.SIP_ERR_CONFIG
    assert b"2^32" in L.sip_last_error(None)


def load_cases():
    with open(os.path.join(GOLD, "ref_tables.json")) as f:
        return json.load(f)["cases"]


@pytest.mark.parametrize("case", load_cases(), ids=lambda c: f"{c['grid']}-{c['blocks_p']}-r{c['ranks']}")
def test_halo_plan_matches_reference_tables(case):
    """sip_plan_halo == the face entries of bsfv::build_transfer_tables, per rank,
    in the reference's canonical order (proj/src/transfers.cpp:148-165)."""
    rank_of = [b[6] for b in case["blocks"]]
    for r, ref in enumerate(case["ranks"]):
        got = sip.plan_halo(case["grid"], case["blocks_p"], rank_of, r)
        assert got.tolist() == ref, f"rank {r}"


def test_halo_plan_send_recv_bijection():
    g, p = (24, 20, 16), (3, 2, 2)
    nb = 12
    for nranks in (1, 2, 3, 4, 6, 12):
        br = sip.plan_block_ranks(p, nranks)
        sends, recvs = [], []
        for r in range(nranks):
            for e in sip.plan_halo(g, p, br, r).tolist():
                if e[0] == 1:
                    sends.append((r, e[3], e[4], e[5], e[2]))
                elif e[0] == 2:
                    recvs.append((e[3], r, e[5], e[4], e[2] ^ 1))
        assert sorted(sends) == sorted(recvs)
        assert all(br[b] in range(nranks) for b in range(nb))


@pytest.mark.parametrize("p,n,expect", [
    ((2, 2, 2), 1, [8]),
    ((4, 2, 2), 2, [8, 8]),
    ((4, 4, 4), 8, [8] * 8),
    ((4, 4, 8), 8, [16] * 8),
])
def test_compact_block_rank_placement(p, n, expect):
    br = sip.plan_block_ranks(p, n)
    counts = [br.count(r) for r in range(n)]
    assert counts == expect
    # each rank owns a compact box of blocks (not with_ranks' slabs)
    px, py, pz = p
    for r in range(n):
        cs = [(b % px, (b // px) % py, b // (px * py)) for b in range(px * py * pz) if br[b] == r]
        ext = [max(c[a] for c in cs) - min(c[a] for c in cs) + 1 for a in range(3)]
        assert ext[0] * ext[1] * ext[2] == len(cs)


def test_config3_gets_2x2x2_per_gpu():
    for world, lat in ((1, (2, 2, 2)), (2, (4, 2, 2)), (4, (4, 4, 2)), (8, (4, 4, 4))):
        br = sip.plan_block_ranks(lat, world)
        px, py, pz = lat
        for r in range(world):
            cs = [(b % px, (b // px) % py, b // (px * py)) for b in range(px * py * pz) if br[b] == r]
            ext = [max(c[a] for c in cs) - min(c[a] for c in cs) + 1 for a in range(3)]
            assert ext == [2, 2, 2]
