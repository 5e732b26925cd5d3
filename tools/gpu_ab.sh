# A/B of a source change: usage bash tools/gpu_ab.sh <file in csrc> <old copy> ; kernel times of one C3 and one C4 view
f=$1; old=$2
cp paper_2411_16392_b200/csrc/$f /tmp/new_$f
run() {
  python -c "from paper_2411_16392_b200 import build as b; b.build(force=True)" > /tmp/build.log 2>&1 || { echo "build failed"; tail -5 /tmp/build.log; }
  for cfg in c3 c4; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file /tmp/l.csv python tools/profile_view.py --config $cfg > /dev/null 2>&1
  python - "$1 $cfg" <<'PY'
import csv, sys, collections
rows=[r for r in csv.reader(open('/tmp/l.csv')) if len(r)>5]
h=rows[0]; ki=h.index('Kernel Name'); vi=h.index('Metric Value')
agg=collections.defaultdict(float)
for r in rows[1:]:
    try: agg[r[ki].split('(')[0]]+=float(r[vi].replace(',',''))/1e6
    except: pass
print(sys.argv[1], {k.split('::')[-1]: round(v,3) for k,v in sorted(agg.items(), key=lambda x:-x[1])[:5]})
PY
  done
}
run new
cp $old paper_2411_16392_b200/csrc/$f; run old
cp /tmp/new_$f paper_2411_16392_b200/csrc/$f; run new
