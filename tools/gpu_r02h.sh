# float64 termination decision: parity (count flips), event count, A/B cost
mkdir -p gpurun_out
python -m paper_2411_16392_b200.build > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_known_answers.py tests/test_debug_checks.py -q -x 2>&1 | tail -2
QGS_PARITY_OUT=gpurun_out/r02h_parity timeout 900 python -m pytest tests/test_gpu_fullview.py -q -x 2>&1 | tail -2
for c in c3 c4; do python -c "
import json; d=json.load(open('gpurun_out/r02h_parity/fullview_$c.json'))
print('$c', d['image'], d['grads'].get('violations'), d['grads'].get('conditioning',{}).get('count_flip'))"; done
QGS_BUILD_DEBUG=0 QGS_NVCC_EXTRA="-DQGS_UTIL_COUNTERS=1" python -c "from paper_2411_16392_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
python tools/lane_util_fwd.py --config c3 | head -1
python tools/lane_util_fwd.py --config c4 | head -1
bash tools/gpu_wpc.sh "" "-DQGS_TERM_BAND=-1.0"
