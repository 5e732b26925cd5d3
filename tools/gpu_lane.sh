# forward lane utilisation (diagnostics build), C3 and C2
QGS_NVCC_EXTRA=-DQGS_UTIL_COUNTERS=1 python -c "from paper_2411_16392_b200 import build as b; b.build(force=True)" > /dev/null 2>&1 || echo "build failed"
timeout 600 python tools/lane_util_fwd.py --config c3 2>&1 | tail -6
timeout 600 python tools/lane_util_fwd.py --config c4 2>&1 | tail -6
