mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02a_smi.txt
lscpu > gpurun_out/r02a_lscpu.txt 2>&1
(time timeout 900 python -m pytest tests -m gpu -x -q) > gpurun_out/r02a_tests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/r02a_tests.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/r02a_bench.log 2>&1; echo "bench rc=$?"
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --exact > gpurun_out/r02a_bench_exact.log 2>&1; echo "bench exact rc=$?"
tail -1 gpurun_out/r02a_bench.log | cut -c1-400
tail -1 gpurun_out/r02a_bench_exact.log | cut -c1-400
