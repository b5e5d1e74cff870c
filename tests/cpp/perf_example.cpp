// The B200 perf header (include/bsfv_perf.hpp) over the shared scenarios of
// oracle/perf_scenario.inc; compared byte for byte with the reference's
// output (tests/golden/perf_golden.txt) by tests/test_perf_report.py.
#include "bsfv_perf.hpp"

using namespace bsfv::b200;
#include "perf_scenario.inc"

int main() { return run_scenarios(std::cin); }
