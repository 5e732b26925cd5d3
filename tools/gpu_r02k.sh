mkdir -p gpurun_out/r02k
(time QGS_PARITY_OUT=gpurun_out/r02k timeout 1500 python -m pytest tests -m gpu -q -rf) > gpurun_out/r02k_tests.log 2>&1; echo "tests rc=$?"
tail -4 gpurun_out/r02k_tests.log
timeout 900 python bench.py > gpurun_out/r02k_bench.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/r02k_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('value',d['value'],'e2e',d['e2e']['value'],'fwd',r['fwd_ms_per_step']/8,'bwd',r['bwd_ms_per_step']/8, 'frac', r['frac'], 'cpu', d['cpu_baseline']['value'], d['cpu_baseline']['sample'])"
