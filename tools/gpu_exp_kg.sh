for flags in "$@"; do
  QGS_NVCC_EXTRA="$flags" python -c "from paper_2411_16392_b200 import build as b; b.build(force=True)" > /dev/null 2>&1 || echo "build failed: $flags"
  echo "== $flags"; python tools/kg_xy_diff.py 2>&1 | head -3
done
