# stream-priority experiment: device-timed C3 bench, default / side high / raster high
python -m paper_2411_16392_b200.build > /dev/null 2>&1
for v in "" "QGS_SIDE_PRIORITY=-5" "QGS_MAIN_PRIORITY=-5" ""; do
  env $v timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1]); r=d['roofline']
print('$v'.ljust(24), round(d['value'],2), 'ms/step', round(d['ms_per_step'],2), 'fwd_pipe', round(r['fwd_ms_per_step_in_pipeline'],2), 'bwd_pipe', round(r['bwd_ms_per_step_in_pipeline'],2), d['clocks'])"
done
