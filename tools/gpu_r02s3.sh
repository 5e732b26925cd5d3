# sort path statistics (C3, C4) + one full ncu capture of the tile sort with source
mkdir -p gpurun_out/s3
python -m paper_2411_16392_b200.build > /dev/null 2>&1
timeout 600 python tools/sort_stats.py --config c3 2>&1 | tail -12
timeout 600 python tools/sort_stats.py --config c4 2>&1 | tail -12
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tile_sort_kernel|pair_key" -c 2 \
  -o gpurun_out/s3/sort_full python tools/profile_view.py --config c3 > gpurun_out/s3/ncu.log 2>&1; echo "ncu rc=$?"
