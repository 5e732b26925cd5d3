mkdir -p gpurun_out/r02u
timeout 1500 python tools/parity_report.py --scenes golden,c1,c2,c5 --views 1 --out gpurun_out/r02u/parity_golden_c1_c2_c5.json > gpurun_out/r02u/parity.log 2>&1; echo "parity rc=$?"
for c in c1 c2 c4 c5; do
  st=5; [ $c = c4 ] && st=3
  timeout 900 python bench.py --config $c --steps $st --warmup 3 --no-cpu > gpurun_out/r02u/bench_$c.log 2>&1; echo "bench $c rc=$?"
  tail -1 gpurun_out/r02u/bench_$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', 'value %.2f e2e %.2f ms %.1f' % (d['value'], d['e2e']['value'], d['ms_per_step']))"
done
