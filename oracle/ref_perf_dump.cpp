// ref_perf_dump.cpp -- TEST INFRASTRUCTURE: the reference's perf module
// (proj/src/perf.cpp, compiled in place from /root/reference; oracle/Makefile
// target `ref`) run over the scenarios of oracle/perf_scenario.inc.  Its output
// is committed as tests/golden/perf_golden.txt (oracle/make_golden.py).
#include "bsfv/perf.hpp"

using namespace bsfv;
#include "perf_scenario.inc"

int main() { return run_scenarios(std::cin); }
