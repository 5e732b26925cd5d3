# usage: CFGS="c3 c4" bash tools/gpu_exp_cfg.sh "<extra nvcc flags>" ... : per variant and config, kernel times of one view
for flags in "$@"; do
  QGS_NVCC_EXTRA="$flags" python -c "from paper_2411_16392_b200 import build as b; b.build(force=True)" > /dev/null 2>&1 || echo "build failed: $flags"
  for CFG in ${CFGS:-c3 c4}; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file /tmp/l.csv python tools/profile_view.py --config $CFG > /dev/null 2>&1
  python - "$flags" "$CFG" <<'PY'
import csv, sys, collections
rows=[r for r in csv.reader(open('/tmp/l.csv')) if len(r)>5]
h=rows[0]; ki=h.index('Kernel Name'); vi=h.index('Metric Value')
agg=collections.defaultdict(float)
for r in rows[1:]:
    try: agg[r[ki].split('(')[0]]+=float(r[vi].replace(',',''))/1e6
    except: pass
print(repr(sys.argv[1]), sys.argv[2], {k.split('::')[-1]: round(v,3) for k,v in sorted(agg.items(), key=lambda x:-x[1]) if "sort" in k or "key" in k})
PY
  done
done
