# Round profiling recipe (B200_PROFILING.md): plain bench, launch list, one
# full capture of K2 and K3 at config 1 fp64.  Outputs in gpurun_out/.
set -x
TAG=${TAG:-r1}
python bench.py --steps 5 --warmup 3 > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err; echo bench rc=$?
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --precision f64"
$CMD > gpurun_out/plain_${TAG}.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_${TAG}.csv $CMD > gpurun_out/ncu_launch_${TAG}.log 2>&1; echo launches rc=$?
ncu --set full --clock-control none --import-source on -k regex:k_forward -s 10 -c 1 -o gpurun_out/prof_fwd_${TAG} $CMD > gpurun_out/ncu_fwd_${TAG}.log 2>&1; echo fwd rc=$?
ncu --set full --clock-control none --import-source on -k regex:k_backward -s 10 -c 1 -o gpurun_out/prof_bwd_${TAG} $CMD > gpurun_out/ncu_bwd_${TAG}.log 2>&1; echo bwd rc=$?
