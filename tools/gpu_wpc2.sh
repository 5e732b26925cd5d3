# usage: bash tools/gpu_wpc2.sh "<flags>" ...   like gpu_wpc.sh, plus the candidate funnel
for flags in "$@"; do
  QGS_BUILD_DEBUG=0 QGS_NVCC_EXTRA="$flags" python -c "from paper_2411_16392_b200 import build as b; b.build(force=True)" > /dev/null 2>&1 || echo "build failed: $flags"
  timeout 600 python bench.py --steps 4 --warmup 3 --no-cpu --no-e2e > /tmp/b.log 2>&1 || { echo "bench failed: $flags"; tail -3 /tmp/b.log; continue; }
  tail -1 /tmp/b.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; a=r['algorithmic']; print(repr(sys.argv[1]), 'value %.2f fwd %.3f bwd %.3f conic %.3e coarse %.3e' % (d['value'], r['fwd_ms_per_step']/8, r['bwd_ms_per_step']/8, a['after_conic_cull'], a['after_coarse_test']))" "$flags"
done
