CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --precision ${PREC:-f64}"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:${KERN:-k_forward} -s 10 -c 1 -o gpurun_out/${OUT:-prof_fwd} $CMD > gpurun_out/ncu_full.log 2>&1; echo full rc=$?
