for f in "" "-DQGS_TERM_BAND=1e-30" "-DQGS_TERM_NOP=1" "-DQGS_TERM_BAND=-1.0"; do
  QGS_BUILD_DEBUG=0 QGS_NVCC_EXTRA="$f" python -c "from paper_2411_16392_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
  echo "== $f"; timeout 300 python tools/term_debug.py c1 s_sh3 2>&1 | grep flips
  timeout 300 python tools/term_debug.py c1 2>&1 | grep flips
done
