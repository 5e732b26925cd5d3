python -m paper_2411_16392_b200.build > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_known_answers.py tests/test_debug_checks.py -q 2>&1 | grep -E "FAILED|passed|failed" | head -20
echo "== counters build"
QGS_BUILD_DEBUG=0 QGS_NVCC_EXTRA="-DQGS_UTIL_COUNTERS=1" python -m paper_2411_16392_b200.build > /dev/null 2>&1
timeout 300 python tools/term_debug.py c1 s_sh3 2>&1 | grep flips
python tools/lane_util_fwd.py --config c3 | head -2
bash tools/gpu_wpc.sh "-DQGS_TERM_BAND=2e-5" "-DQGS_TERM_BAND=-1.0" "-DQGS_TERM_BAND=1e-4"
