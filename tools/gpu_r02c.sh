mkdir -p gpurun_out/r02c
(time QGS_PARITY_OUT=gpurun_out/r02c timeout 1500 python -m pytest tests -m gpu -q -rf --durations=10) > gpurun_out/r02c_tests.log 2>&1; echo "tests rc=$?"
tail -15 gpurun_out/r02c_tests.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/r02c_bench.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/r02c_bench.log | cut -c1-300
