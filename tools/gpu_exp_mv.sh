# usage: bash tools/gpu_exp_mv.sh "<flags>" ... : multiview kernel time per variant (bench_aux)
for flags in "$@"; do
  QGS_NVCC_EXTRA="$flags" python -c "from paper_2411_16392_b200 import build as b; b.build(force=True)" > /dev/null 2>&1 || echo "build failed: $flags"
  python tools/bench_aux.py --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(repr('$flags'), 'multiview_ms', round(d['multiview_ms'], 3))"
done
