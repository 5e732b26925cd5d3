mkdir -p gpurun_out/r02t
(QGS_PARITY_OUT=gpurun_out/r02t timeout 1500 python -m pytest tests -m gpu -q -rf) > gpurun_out/r02t_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r02t_tests.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
bash tools/round_profile.sh r02c
tail -1 gpurun_out/r02c_bench.log | cut -c1-300
