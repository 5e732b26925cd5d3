set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r1_tests.log 2>&1; echo "tests rc=$?"
tail -5 gpurun_out/r1_tests.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/r1_bench.log 2>&1; echo "bench rc=$?"
tail -2 gpurun_out/r1_bench.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1_launches.csv python tools/profile_view.py --config c3 > gpurun_out/r1_ncu_launch.log 2>&1; echo "ncu1 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:raster_ -c 2 -o gpurun_out/r1_raster python tools/profile_view.py --config c3 > gpurun_out/r1_ncu_full.log 2>&1; echo "ncu2 rc=$?"
