# A/B: build with the given WB values and bench each (fwd ms per view from the launch list)
for wb in "$@"; do
  sed -i "s/^constexpr int WB = [0-9]*;/constexpr int WB = $wb;/" paper_2411_16392_b200/csrc/raster_warp.cu
  python -c "from paper_2411_16392_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
  timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('WB=$wb', d['value'], r['fwd_ms_per_step'], r['bwd_ms_per_step'])"
done
