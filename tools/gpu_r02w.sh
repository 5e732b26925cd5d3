for flags in "" "-DQGS_PRE_MIN_BLOCKS=4 -DQGS_CHAIN_MIN_BLOCKS=4" "-DQGS_PRE_MIN_BLOCKS=3 -DQGS_CHAIN_MIN_BLOCKS=3"; do
  QGS_BUILD_DEBUG=0 QGS_NVCC_EXTRA="$flags" python -c "from paper_2411_16392_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file /tmp/l4.csv -k regex:"preprocess|chain" python tools/profile_view.py --config c4 > /dev/null 2>&1
  python - "$flags" <<'PY'
import csv, collections, sys
rows=[r for r in csv.reader(open('/tmp/l4.csv')) if len(r)>5]
h=rows[0]; ki=h.index('Kernel Name'); vi=h.index('Metric Value')
agg=collections.defaultdict(float)
for r in rows[1:]:
    try: agg[r[ki].split('(')[0]]+=float(r[vi].replace(',',''))/1e6
    except: pass
print(repr(sys.argv[1]), {k.split('::')[-1]: round(v,3) for k,v in agg.items()})
PY
done
