QGS_BUILD_DEBUG=0 QGS_NVCC_EXTRA="-DQGS_UTIL_COUNTERS=1" python -c "from paper_2411_16392_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
python tools/lane_util_fwd.py --config c3
python tools/lane_util_fwd.py --config c4
python tools/lane_util_fwd.py --config c5
