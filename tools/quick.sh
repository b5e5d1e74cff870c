# quick GPU check: parity tests + short bench summary
timeout 400 python -m pytest tests/test_gpu_parity.py -q -m gpu --timeout 120 -x > gpurun_out/pytest_q.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_q.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu ${BENCH_ARGS} > gpurun_out/bench_q.log 2>&1; echo bench rc=$?
tail -1 gpurun_out/bench_q.log | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('f64 MLUP/s %.0f fwd %.3f ms bwd %.3f ms frac_step %.3f e2e %.0f' % (d['value'], d['roofline']['launch_ms'], d['k3_backward']['launch_ms'], d['achieved_frac_step'], d['e2e']['value'] if d['e2e'] else 0))
if 'f32' in d: print('f32 MLUP/s %.0f fwd %.3f ms bwd %.3f ms frac_step %.3f' % (d['f32']['value'], d['f32']['roofline']['launch_ms'], d['f32']['k3_backward']['launch_ms'], d['f32']['achieved_frac_step']))
" || tail -20 gpurun_out/bench_q.log
