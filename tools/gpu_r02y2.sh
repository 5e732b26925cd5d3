QGS_BUILD_DEBUG=0 QGS_NVCC_EXTRA="-DQGS_KEY_PAIR2=1" python -m paper_2411_16392_b200.build > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "bin or key or sort or dup" 2>&1 | tail -1
bash tools/gpu_launch_cmp.sh "" "-DQGS_KEY_PAIR2=1" 2>&1 | sed 's/.raster_[a-z_]*kernel.: [0-9.]*, //g'
