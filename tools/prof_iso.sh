#!/bin/bash
# ncu source-level capture of one isolated-brick K2 and K3 launch (f64 by
# default) -> gpurun_out/k{2,3}iso.ncu-rep; run under tools/gpu.sh
P=${1:-f64}; G=${2:-8x32x256}
for K in k_backward:k3iso k_forward:k2iso; do
  ncu --set full --import-source on --clock-control none --warp-sampling-interval 0 -k regex:${K%%:*} -s 4 -c 1 \
      -o gpurun_out/${K##*:} -f python tools/sweep_time.py $P $G 5 > gpurun_out/${K##*:}.log 2>&1
done
