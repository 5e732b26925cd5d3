python -m paper_2411_16392_b200.build > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "cull" 2>&1 | tail -1
bash tools/gpu_wpc2.sh "" "-DQGS_CONIC_LAM_OPT=0" ""
