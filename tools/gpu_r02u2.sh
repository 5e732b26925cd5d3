python -m paper_2411_16392_b200.build > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_known_answers.py -q 2>&1 | tail -1
bash tools/gpu_wpc.sh "" "-DQGS_RED_UNROLL4=1" "" "-DQGS_RED_UNROLL4=1"
