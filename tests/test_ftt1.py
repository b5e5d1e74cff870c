"""FTT1 transfer-table ingest: the library's reader,
writer and send/recv validator against files written by the reference's own
write_tables and against the reference reader's / validator's messages on
corrupted copies (golden: tests/golden/ftt1/, oracle/make_golden.py, the
reference compiled in place).  CPU only (the C-ABI functions are host code)."""
import importlib.util
import json
import os

import numpy as np
import pytest

import paper_1303_4538_b200 as sip

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden", "ftt1")
with open(os.path.join(GOLD, "cases.json")) as f:
    CASES = json.load(f)
_spec = importlib.util.spec_from_file_location("mg", os.path.join(ROOT, "oracle", "make_golden.py"))
_mg = importlib.util.module_from_spec(_spec)
_spec.loader.exec_module(_mg)


def _bytes(name):
    with open(os.path.join(GOLD, name + ".ftt1"), "rb") as f:
        return f.read()


@pytest.mark.parametrize("name", sorted(CASES["files"]))
def test_read_write_validate_reference_files(name):
    data = _bytes(name)
    tables = sip.ftt1_read(data)
    gold = CASES["files"][name]["entries"]
    assert len(tables) == len(gold)
    for t, g in zip(tables, gold):
        assert t.tolist() == g
    assert sip.ftt1_write(tables) == data  # byte-identical round trip
    sip.ftt1_validate(tables)


@pytest.mark.parametrize("name", sorted(CASES["corrupt"]))
def test_corruptions_match_reference_messages(name):
    c = CASES["corrupt"][name]
    data = _mg.ftt1_corrupt(_bytes(c["base"]), c["edit"])
    if c["read"] != "ok":
        with pytest.raises(sip.FormatError) as e:
            sip.ftt1_read(data)
        assert str(e.value) == c["read"][len("error: "):]
        assert e.value.offset == int(c["read"].rsplit(" ", 1)[1].rstrip(")"))
        return
    tables = sip.ftt1_read(data)
    if c["validate"] == "ok":
        sip.ftt1_validate(tables)
    else:
        with pytest.raises(sip.ProtocolError) as e:
            sip.ftt1_validate(tables)
        assert str(e.value) == c["validate"][len("error: "):]


def test_plan_halo_equals_reference_face_entries():
    """The built-in plan (sip_plan_halo_periodic) is the face subset of the
    reference's table, wall and periodic decompositions alike (periodic wraps,
    px = 1 self-wraps, transfers.cpp:15-25 and its canonical order)."""
    for name, f in CASES["files"].items():
        tables = sip.ftt1_read(_bytes(name))
        nr = len(tables)
        br = [int(x) for x in _rank_of_blocks(tables, f["p"])]
        for r in range(nr):
            mine = sip.plan_halo(f["g"], f["p"], br, r, f["periodic_mask"]).tolist()
            ref = [row for row in tables[r].tolist() if row[1] == 0]
            assert mine == ref, (name, r)


def _rank_of_blocks(tables, p):
    nb = p[0] * p[1] * p[2]
    out = [0] * nb
    for r, t in enumerate(tables):
        for row in t.tolist():
            if row[0] != 2:  # local / send: owner is on rank r
                out[row[4]] = r
    return out


CPP_SRC = r'''
#include <cstdio>
#include <fstream>
#include <iterator>
#include "bsfv_sip.hpp"
using namespace bsfv::b200;
int main(int argc, char** argv) {
  std::ifstream f(argv[1], std::ios::binary);
  std::vector<unsigned char> img((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
  TableRows t = read_tables(img);
  validate_matching(t);
  std::printf("ranks %zu entries %zu roundtrip %d\n", t.size(), t[0].size(), (int)(write_tables(t) == img));
  std::vector<unsigned char> cut(img.begin(), img.begin() + 18);
  try { read_tables(cut); } catch (const FormatError& e) { std::printf("format %zu %s\n", e.offset(), e.what()); }
  t[0][0][3] = 1;
  try { validate_matching(t); } catch (const ProtocolError& e) { std::printf("protocol %s\n", e.what()); }
  return 0;
}
'''


def test_cpp_shim_tables(tmp_path):
    import subprocess
    src = tmp_path / "tables.cpp"
    src.write_text(CPP_SRC)
    exe = str(tmp_path / "tables")
    libdir = os.path.join(ROOT, "paper_1303_4538_b200")
    subprocess.run(["g++", "-std=c++17", "-I", os.path.join(ROOT, "include"), str(src), "-o", exe,
                    os.path.join(libdir, "libsip_b200.so"), "-Wl,-rpath," + libdir],
                   check=True, capture_output=True)
    out = subprocess.run([exe, os.path.join(GOLD, "wall_2x2x1_r2.ftt1")], capture_output=True,
                         text=True, check=True).stdout.splitlines()
    n0 = len(CASES["files"]["wall_2x2x1_r2"]["entries"][0])
    assert out[0] == f"ranks 2 entries {n0} roundtrip 1"
    assert out[1] == ("format 16 transfer table file truncated reading entry count "
                      "(at byte offset 16)")
    assert out[2] == "protocol rank 0 has a local entry with peer 1"
