# usage: bash tools/round_summarize.sh TAG  (here, after round_profile.sh ran on the GPU box)
TAG=${1:-r02}
set -e
tail -1 gpurun_out/${TAG}_bench.log > profiles/${TAG}_bench_c3.json
python tools/ncu_summary.py gpurun_out/${TAG}_full.ncu-rep . --json profiles/${TAG}_traffic.json > profiles/${TAG}_ncu_summary.txt
python tools/ncu_lines.py gpurun_out/${TAG}_full.ncu-rep raster_fwd 60 > profiles/${TAG}_ncu_raster_fwd_lines.txt
python tools/ncu_lines.py gpurun_out/${TAG}_full.ncu-rep raster_bwd 60 > profiles/${TAG}_ncu_raster_bwd_lines.txt
python tools/launch_summary.py gpurun_out/${TAG}_launches.csv > profiles/${TAG}_launches_summary.txt
cp gpurun_out/${TAG}_launches.csv profiles/${TAG}_launches.csv
ls -la profiles/ | grep ${TAG}
