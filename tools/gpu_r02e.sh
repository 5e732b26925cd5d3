mkdir -p gpurun_out/r02e
(time QGS_PARITY_OUT=gpurun_out/r02e timeout 900 python -m pytest tests/test_gpu_fullview.py tests/test_gpu_parity.py -q -rf -x) > gpurun_out/r02e_tests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/r02e_tests.log
for i in 1 2; do timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/r02e_bench$i.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/r02e_bench$i.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('value',d['value'],'fwd',r['fwd_ms_per_step']/8,'bwd',r['bwd_ms_per_step']/8)"; done
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --fp32-decisions > gpurun_out/r02e_bench_fp32.log 2>&1
tail -1 gpurun_out/r02e_bench_fp32.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('fp32 value',d['value'],'fwd',r['fwd_ms_per_step']/8,'bwd',r['bwd_ms_per_step']/8)"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02e_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1; echo "ncu rc=$?"
python tools/launch_summary.py gpurun_out/r02e_launches.csv | head -20
