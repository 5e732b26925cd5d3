bash tools/gpu_wpc.sh "" "-DQGS_NEWTON_BAL=1" "-DQGS_EVAL_RSQRT=1" "" "-DQGS_NEWTON_BAL=1" "-DQGS_EVAL_RSQRT=1"
