# flat pair-key kernel: bit-exactness tests, then A/B against the warp-per-primitive kernel
mkdir -p gpurun_out
QGS_BUILD_DEBUG=0 python -c "from paper_2411_16392_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_known_answers.py -q -x 2>&1 | tail -3
QGS_PARITY_OUT=gpurun_out/r02f_parity timeout 900 python -m pytest tests/test_gpu_fullview.py -q -x 2>&1 | tail -2
bash tools/gpu_launch_cmp.sh "" "-DQGS_KEY_FLAT=0"
bash tools/gpu_wpc.sh "" "-DQGS_KEY_FLAT=0"
