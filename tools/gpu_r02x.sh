bash tools/gpu_wpc.sh "" "-DQGS_NEWTON_F32_FIRST=1"
QGS_BUILD_DEBUG=0 QGS_NVCC_EXTRA="-DQGS_NEWTON_F32_FIRST=1" python -c "from paper_2411_16392_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
mkdir -p gpurun_out/r02x
QGS_PARITY_OUT=gpurun_out/r02x timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_known_answers.py tests/test_gpu_fullview.py -q -rf 2>&1 | tail -3
