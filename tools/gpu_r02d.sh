# final round-2 validation: full GPU suite, smoke, bench + profiles (tag r02d)
mkdir -p gpurun_out
QGS_PARITY_OUT=gpurun_out/r02d_parity timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r02d_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r02d_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02d_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r02d_smoke.log
bash tools/round_profile.sh r02d
tail -1 gpurun_out/r02d_bench.log | cut -c1-400
