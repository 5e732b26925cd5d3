# float64 termination: which test failed, and the error distribution of T at the events
mkdir -p gpurun_out
python -m paper_2411_16392_b200.build > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_known_answers.py tests/test_debug_checks.py -q 2>&1 | grep -E "FAILED|passed|failed|Error|assert" | head -20
QGS_BUILD_DEBUG=0 QGS_NVCC_EXTRA="-DQGS_UTIL_COUNTERS=1" python -c "from paper_2411_16392_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
for c in c3 c4 c2 c5; do python tools/lane_util_fwd.py --config $c | head -2; done
