# usage: bash tools/gpu_check.sh TAG  -- gpu tests + bench (+ launch list)
TAG=${1:-x}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_tests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/${TAG}_tests.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/${TAG}_bench.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/${TAG}_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('value',d['value'],'ms',d['ms_per_step'],'fwd',r['fwd_ms_per_step'],'bwd',r['bwd_ms_per_step'],'e2e',d.get('e2e',{}).get('value'))"
if [ "$2" = "ncu" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv python tools/profile_view.py --config c3 > /dev/null 2>&1; echo "ncu rc=$?"
fi
