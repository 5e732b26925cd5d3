# round-2 final (after the latency-chain work): full GPU suite, smoke, bench + profiles (tag r02g)
mkdir -p gpurun_out
python -m paper_2411_16392_b200.build > /dev/null 2>&1
QGS_PARITY_OUT=gpurun_out/r02g_parity timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02g_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r02g_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02g_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r02g_smoke.log
bash tools/round_profile.sh r02g
tail -1 gpurun_out/r02g_bench.log | cut -c1-300
