mkdir -p gpurun_out/r02q
(QGS_PARITY_OUT=gpurun_out/r02q timeout 1500 python -m pytest tests -m gpu -q -rf -x) > gpurun_out/r02q_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r02q_tests.log
for c in c3 c4 c5; do
  st=4; [ $c = c4 ] && st=2
  timeout 900 python bench.py --config $c --steps $st --warmup 3 --no-cpu --no-e2e > /tmp/b.log 2>&1
  tail -1 /tmp/b.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; V=d['config']['views_per_step']; print('$c value %.2f fwd %.3f bwd %.3f' % (d['value'], r['fwd_ms_per_step']/V, r['bwd_ms_per_step']/V))"
done
