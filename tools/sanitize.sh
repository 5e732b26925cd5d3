# usage: bash tools/sanitize.sh OUTDIR -- compute-sanitizer memcheck / racecheck / synccheck /
# initcheck over tools/sanitize_view.py (C1: 2048 primitives, 128x128)
OUT=${1:-gpurun_out/sanitize}
mkdir -p $OUT
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ "$tool" = "racecheck" ] && extra="--racecheck-report all"
  timeout 1200 compute-sanitizer --tool $tool $extra --print-limit 50 \
     --kernel-name regex:qgs \
     python tools/sanitize_view.py > $OUT/$tool.log 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' $OUT/$tool.log | tail -1)"
done
