timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullview.py -q -x -k "scale or sort or binning or c4" 2>&1 | tail -2
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file /tmp/l4.csv python tools/profile_view.py --config c4 > /dev/null 2>&1
python - <<'PY'
import csv, collections
rows=[r for r in csv.reader(open('/tmp/l4.csv')) if len(r)>5]
h=rows[0]; ki=h.index('Kernel Name'); vi=h.index('Metric Value')
agg=collections.defaultdict(float)
for r in rows[1:]:
    try: agg[r[ki].split('(')[0]]+=float(r[vi].replace(',',''))/1e6
    except: pass
print('c4 view', {k.split('::')[-1]: round(v,3) for k,v in sorted(agg.items(), key=lambda x:-x[1])[:8]})
PY
timeout 900 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu --no-e2e > /tmp/b.log 2>&1; tail -1 /tmp/b.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c4 value %.2f' % d['value'])"
timeout 900 python bench.py --steps 4 --warmup 3 --no-cpu --no-e2e > /tmp/b.log 2>&1; tail -1 /tmp/b.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3 value %.2f' % d['value'])"
