python -m paper_2411_16392_b200.build > /dev/null 2>&1
timeout 600 python tools/term_debug.py 2>&1 | tail -60
