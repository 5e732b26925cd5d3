# flat pair-key kernel, software-pipelined: bit-exactness, then per-kernel A/B
mkdir -p gpurun_out
QGS_BUILD_DEBUG=0 python -c "from paper_2411_16392_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "bin or key or sort or golden" 2>&1 | tail -2
bash tools/gpu_launch_cmp.sh "" "-DQGS_KEY_MIN_BLOCKS=3" "-DQGS_KEY_FLAT=0" 2>&1 | sed 's/raster_[a-z_]*kernel[^,]*,//g'
grep -h key_rec /tmp/l.csv | head -0
