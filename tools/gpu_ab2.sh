python -m paper_2411_16392_b200.build > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "binning or sort" 2>&1 | tail -1
bash tools/gpu_ab.sh binning.cu tools/ab/binning_old.cu
mkdir -p gpurun_out/s4
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tile_sort_kernel" -c 1 \
  -o gpurun_out/s4/sort_full python tools/profile_view.py --config c3 > gpurun_out/s4/ncu.log 2>&1; echo "ncu rc=$?"
