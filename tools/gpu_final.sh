# last check of the round's final commit: full GPU suite, smoke, default bench
mkdir -p gpurun_out
python -m paper_2411_16392_b200.build > /dev/null 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/final_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/final_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/final_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/final_bench.log | cut -c1-200
