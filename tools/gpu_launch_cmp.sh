# usage: bash tools/gpu_launch_cmp.sh "<flags>" ... : per-kernel ms of one C3 view per variant
for flags in "$@"; do
  QGS_BUILD_DEBUG=0 QGS_NVCC_EXTRA="$flags" python -c "from paper_2411_16392_b200 import build as b; b.build(force=True)" > /dev/null 2>&1 || echo "build failed: $flags"
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file /tmp/l.csv python tools/profile_view.py --config c3 > /dev/null 2>&1
  python - "$flags" <<'PY'
import csv, sys, collections
rows=[r for r in csv.reader(open('/tmp/l.csv')) if len(r)>5]
h=rows[0]; ki=h.index('Kernel Name'); vi=h.index('Metric Value')
agg=collections.defaultdict(float)
for r in rows[1:]:
    try: agg[r[ki].split('(')[0]]+=float(r[vi].replace(',',''))/1e6
    except: pass
print(repr(sys.argv[1]), {k.split('::')[-1]: round(v,3) for k,v in sorted(agg.items(), key=lambda x:-x[1])[:9]})
PY
done
