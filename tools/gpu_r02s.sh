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
