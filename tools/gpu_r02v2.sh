python -m paper_2411_16392_b200.build > /dev/null 2>&1
bash tools/gpu_wpc.sh "" "-DQGS_RED_SETS=16" "-DQGS_BWD_MIN_BLOCKS=16" "-DQGS_BWD_MIN_BLOCKS=24" ""
