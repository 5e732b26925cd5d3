mkdir -p gpurun_out/r02f
(time QGS_PARITY_OUT=gpurun_out/r02f timeout 1500 python -m pytest tests -m gpu -q -rf -x) > gpurun_out/r02f_tests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/r02f_tests.log
for i in 1 2; do timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/r02f_bench$i.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/r02f_bench$i.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('value',d['value'],'fwd',r['fwd_ms_per_step']/8,'bwd',r['bwd_ms_per_step']/8, 'frac', r['frac'])"; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02f_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1; echo "ncu rc=$?"
python tools/launch_summary.py gpurun_out/r02f_launches.csv | head -14
