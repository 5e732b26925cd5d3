mkdir -p gpurun_out
timeout 600 python tools/grad_prim_diag.py --config c4 --prims 1269412 > gpurun_out/r02g_diag.log 2>&1; echo "diag rc=$?"
cat gpurun_out/r02g_diag.log | tail -12
for mb in 16 17 18; do
  QGS_NVCC_EXTRA="-DQGS_FWD_EXACT_MIN_BLOCKS=$mb" python -c "from paper_2411_16392_b200 import build as b; b.build(force=True)" > /dev/null 2>&1 || echo "build failed"
  timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/r02g_mb$mb.log 2>&1
  tail -1 gpurun_out/r02g_mb$mb.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('mb $mb value',d['value'],'fwd',r['fwd_ms_per_step']/8,'bwd',r['bwd_ms_per_step']/8)"
done
