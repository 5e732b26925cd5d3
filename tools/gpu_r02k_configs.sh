# final per-config bench lines + the fp32-decision mode at C3
mkdir -p gpurun_out
python -m paper_2411_16392_b200.build > /dev/null 2>&1
rm -f gpurun_out/r02k_configs.jsonl
for c in c1 c2 c4 c5; do timeout 900 python bench.py --config $c --no-cpu 2>/dev/null | tail -1 >> gpurun_out/r02k_configs.jsonl; done
timeout 600 python bench.py --fp32-decisions --no-cpu --no-e2e 2>/dev/null | tail -1 > gpurun_out/r02k_fp32.json
python - <<'PY'
import json
for l in open('gpurun_out/r02k_configs.jsonl'):
    d = json.loads(l); print(d['config']['workload'][:40], round(d['value'], 1), round(d['e2e']['value'], 1))
d = json.load(open('gpurun_out/r02k_fp32.json')); r = d['roofline']
print('fp32 decisions c3', round(d['value'], 1), 'fwd', round(r['fwd_ms_per_step'] / 8, 3), 'bwd', round(r['bwd_ms_per_step'] / 8, 3))
PY
