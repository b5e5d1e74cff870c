"""Profiling / parallel-efficiency reporting of the B200
framework, include/bsfv_perf.hpp: byte-identical to the reference's own perf
module (proj/src/perf.cpp) on the committed scenarios (golden output made by
oracle/make_golden.py from the reference compiled in place), plus the SPEC's
profile_report examples.  CPU only."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")


def _build(tmp_path, src, extra=()):
    exe = str(tmp_path / os.path.splitext(os.path.basename(src))[0])
    cmd = ["g++", "-O2", "-std=c++17", "-I", os.path.join(ROOT, "include"), "-I",
           os.path.join(ROOT, "oracle"), src, "-o", exe, *extra]
    subprocess.run(cmd, check=True, capture_output=True)
    return exe


def test_efficiency_matches_reference_bytes(tmp_path):
    exe = _build(tmp_path, os.path.join(ROOT, "tests", "cpp", "perf_example.cpp"))
    with open(os.path.join(GOLD, "perf_scenarios.txt")) as f:
        out = subprocess.run([exe], stdin=f, capture_output=True, text=True, check=True).stdout
    with open(os.path.join(GOLD, "perf_golden.txt")) as f:
        gold = f.read()
    assert out == gold


PROFILE_SRC = r'''
#include <cstdio>
#include "bsfv_perf.hpp"
using namespace bsfv::b200;
int main() {
  TimerSet r0, r1;
  r0.add("sip sweep", 3.0, 10); r0.add("halo", 1.0, 10);
  r1.add("sip sweep", 2.5, 10); r1.add("halo", 1.0, 10); r1.add("io", 0.0, 1);
  auto p = profile_report({&r0, &r1});
  std::printf("%s", profile_csv(p).c_str());
  std::printf("%s", profile_table(profile_report({&r0}, 1)).c_str());
  TimerSet one; one.add("solve", 2.0, 1);
  std::printf("%s", profile_csv(profile_report({&one})).c_str());
  TimerSet nest;
  { TimerSet::Scope a(&nest, "outer"); TimerSet::Scope b(&nest, "inner"); }
  std::printf("nested %zu %d\n", nest.records().size(), nest.records().at("outer").self_s >= 0);
  try { nest.exit(); } catch (const MisuseError&) { std::printf("misuse ok\n"); }
  return 0;
}
'''


def test_profile_report_examples(tmp_path):
    src = tmp_path / "profile.cpp"
    src.write_text(PROFILE_SRC)
    out = subprocess.run([_build(tmp_path, str(src))], capture_output=True, text=True,
                         check=True).stdout.splitlines()
    # max over ranks (3.0 s, 1.0 s, 0.0 s), summed calls, 75 % / 25 %
    assert out[:4] == ["name,self_s,calls,pct", "sip sweep,3,20,75", "halo,1,20,25", "io,0,1,0"]
    assert out[4].startswith("time %") and out[5].split() == ["75.00", "3.0000", "10", "sip", "sweep"]
    assert out[6:8] == ["name,self_s,calls,pct", "solve,2,1,100"]  # one region of 2 s -> 100 %
    assert out[8] == "nested 2 1" and out[9] == "misuse ok"
