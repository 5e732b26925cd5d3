mkdir -p gpurun_out/r02i
(time QGS_PARITY_OUT=gpurun_out/r02i timeout 1500 python -m pytest tests -m gpu -q -rf) > gpurun_out/r02i_tests.log 2>&1; echo "tests rc=$?"
tail -4 gpurun_out/r02i_tests.log
for i in 1 2; do timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/r02i_bench$i.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/r02i_bench$i.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('value',d['value'],'fwd',r['fwd_ms_per_step']/8,'bwd',r['bwd_ms_per_step']/8, 'frac', r['frac'], d['fragment_log'])"; done
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --fp32-decisions > gpurun_out/r02i_bench_fp32.log 2>&1
tail -1 gpurun_out/r02i_bench_fp32.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('fp32 value',d['value'],'fwd',r['fwd_ms_per_step']/8,'bwd',r['bwd_ms_per_step']/8)"
