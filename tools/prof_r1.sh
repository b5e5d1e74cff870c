set -x
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --precision f64"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches_r1.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo launches rc=$?
$CMD > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_forward -s 10 -c 1 -o gpurun_out/prof_fwd_r1 $CMD > gpurun_out/ncu_full.log 2>&1; echo full rc=$?
ncu --set full --clock-control none --import-source on -k regex:k_backward -s 10 -c 1 -o gpurun_out/prof_bwd_r1 $CMD > gpurun_out/ncu_full_b.log 2>&1; echo fullb rc=$?
ls -la gpurun_out
