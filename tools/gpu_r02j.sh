mkdir -p gpurun_out
timeout 900 python tools/grad_frag_diag.py --config c4 --prim 1269412 > gpurun_out/r02j_fragdiag.log 2>&1; echo "diag rc=$?"
tail -25 gpurun_out/r02j_fragdiag.log
bash tools/sanitize.sh gpurun_out/r02j_sanitize
