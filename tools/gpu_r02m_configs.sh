# final per-config bench lines at r02m + the reference arm (CPU oracle port) at the driver's defaults
mkdir -p gpurun_out
python -m paper_2411_16392_b200.build > /dev/null 2>&1
rm -f gpurun_out/r02m_configs.jsonl
for c in c1 c2 c4 c5; do timeout 900 python bench.py --config $c --no-cpu 2>/dev/null | tail -1 >> gpurun_out/r02m_configs.jsonl; done
( time timeout 900 python bench.py --impl reference ) 2>&1 | tail -5 > gpurun_out/r02m_reference.log
python - <<'PY'
import json
for l in open('gpurun_out/r02m_configs.jsonl'):
    d = json.loads(l); print(d['config']['workload'][:40], round(d['value'], 1), round(d['e2e']['value'], 1))
PY
cat gpurun_out/r02m_reference.log | cut -c1-400
