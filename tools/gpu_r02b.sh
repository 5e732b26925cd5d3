mkdir -p gpurun_out
(time timeout 1500 python -m pytest tests -m gpu -q -rf --durations=15) > gpurun_out/r02b_tests.log 2>&1; echo "tests rc=$?"
tail -30 gpurun_out/r02b_tests.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/r02b_bench.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/r02b_bench.log | cut -c1-300
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r02b_ref.log 2>&1; echo "ref rc=$?"
tail -1 gpurun_out/r02b_ref.log
