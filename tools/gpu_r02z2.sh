# final-code parity report: goldens + full C1 / C2 / C5 views (default settings)
mkdir -p gpurun_out/r02z
python -m paper_2411_16392_b200.build > /dev/null 2>&1
timeout 1500 python tools/parity_report.py --scenes golden,c1,c2,c5 --views 1 --out gpurun_out/r02z/parity_golden_c1_c2_c5.json > gpurun_out/r02z/parity.log 2>&1; echo "parity rc=$?"
python - <<'PY'
import json
d = json.load(open('gpurun_out/r02z/parity_golden_c1_c2_c5.json'))
for k, v in (d.items() if isinstance(d, dict) else enumerate(d)):
    if isinstance(v, dict):
        im = v.get('image', {}); g = v.get('grads', {})
        print(k, {x: im.get(x) for x in ('count_flip_pixels', 'over_tol_pixels', 'over_tol_same_count')}, 'grad viol', g.get('violations'), 'sort', v.get('binning', v.get('sort')))
PY
