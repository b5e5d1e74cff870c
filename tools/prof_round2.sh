# Round-2 profiling recipe (B200_PROFILING.md), config 1 (256^3):
#   plain bench line; for f64 and f32: the gpu__time_duration launch list of
#   the same bench command, then one ncu --set full capture each of K2 and K3.
# Outputs in gpurun_out/ (summarised into profiles/ by tools/prof_extract.py).
set -x
TAG=${TAG:-r2}
python bench.py --steps 5 --warmup 3 > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err; echo bench rc=$?
for P in f64 f32; do
  CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-caller --no-extra --precision $P"
  $CMD > gpurun_out/plain_${TAG}_$P.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_${TAG}_$P.csv $CMD > gpurun_out/ncu_launch_${TAG}_$P.log 2>&1; echo launches $P rc=$?
  for K in k_forward:fwd k_backward:bwd; do
    ncu --set full --clock-control none --import-source on -k regex:${K%%:*} -s 10 -c 1 \
        -o gpurun_out/prof_${K##*:}_${TAG}_$P -f $CMD > gpurun_out/ncu_${K##*:}_${TAG}_$P.log 2>&1; echo ${K##*:} $P rc=$?
  done
done
