# usage: bash tools/round_profile.sh TAG  (on the GPU box; outputs in gpurun_out/)
TAG=${1:-r02}
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/${TAG}_bench.log 2>&1; echo "bench rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e \
  > gpurun_out/${TAG}_ncu_launch.log 2>&1; echo "launch list rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on \
  -k regex:"raster_fwd|raster_bwd_kernel|tile_sort|pair_key|preprocess|chain" -c 7 -o gpurun_out/${TAG}_full \
  python tools/profile_view.py --config c3 > gpurun_out/${TAG}_ncu_full.log 2>&1; echo "ncu full rc=$?"
