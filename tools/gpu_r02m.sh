python -m paper_2411_16392_b200.build > /dev/null 2>&1
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | grep -E "FAILED|passed|failed" | head -20
echo "== counters build (no other change)"
QGS_BUILD_DEBUG=0 QGS_NVCC_EXTRA="-DQGS_UTIL_COUNTERS=1" python -m paper_2411_16392_b200.build > /dev/null 2>&1
timeout 300 python tools/term_debug.py c1 s_sh3 s_default 2>&1 | grep flips
