# usage: bash tools/gpu_exp_aux.sh "<flags>" ... : aux kernel times per build variant (bench_aux)
for flags in "$@"; do
  QGS_NVCC_EXTRA="$flags" python -c "from paper_2411_16392_b200 import build as b; b.build(force=True)" > /dev/null 2>&1 || echo "build failed: $flags"
  python tools/bench_aux.py --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(repr('$flags'), {k: round(v, 3) for k, v in d.items() if k.endswith('_ms') or k.endswith('_frac')})"
done
