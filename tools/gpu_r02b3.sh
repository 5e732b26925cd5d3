python -m paper_2411_16392_b200.build > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q 2>&1 | tail -1
QGS_PARITY_OUT=gpurun_out/b3 timeout 900 python -m pytest tests/test_gpu_fullview.py -q -k c4 2>&1 | tail -1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file /tmp/l3.csv python tools/profile_view.py --config c3 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file /tmp/l4.csv python tools/profile_view.py --config c4 > /dev/null 2>&1
for f in /tmp/l3.csv /tmp/l4.csv; do python - "$f" <<'PY'
import csv, sys, collections
rows=[r for r in csv.reader(open(sys.argv[1])) if len(r)>5]
h=rows[0]; ki=h.index('Kernel Name'); vi=h.index('Metric Value')
agg=collections.defaultdict(float)
for r in rows[1:]:
    try: agg[r[ki].split('(')[0]]+=float(r[vi].replace(',',''))/1e6
    except: pass
print(sys.argv[1], {k.split('::')[-1]: round(v,3) for k,v in agg.items() if 'sort' in k})
PY
done
