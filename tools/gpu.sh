#!/bin/bash
# Local wrapper: rebuild the in-tree .so (abort on failure), then run the
# given command on a B200 via gpurun.  Usage: tools/gpu.sh <timeout_s> '<cmd>'
set -e
make -s -C /root/repo/paper_1303_4538_b200/csrc >/dev/null || { echo "BUILD FAILED"; exit 1; }
make -s -C /root/repo/oracle >/dev/null
T=${1:-600}; shift
exec /usr/local/graft/bin/gpurun --timeout "$T" -- "$@"
