QGS_BUILD_DEBUG=0 QGS_NVCC_EXTRA="-DQGS_UTIL_COUNTERS=1" python -c "from paper_2411_16392_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
python tools/lane_util_fwd.py --config c3
python tools/lane_util_fwd.py --config c4
for flags in "" "-DQGS_FWD_WPC=1"; do
  QGS_BUILD_DEBUG=0 QGS_NVCC_EXTRA="$flags" python -c "from paper_2411_16392_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
  for mode in "" "--fp32-decisions"; do
    timeout 900 python bench.py --config c4 --steps 2 --warmup 3 --no-cpu --no-e2e $mode > /tmp/b.log 2>&1
    tail -1 /tmp/b.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(repr('$flags'), '$mode', 'c4 value %.2f fwd %.3f bwd %.3f' % (d['value'], r['fwd_ms_per_step']/64, r['bwd_ms_per_step']/64))"
  done
done
