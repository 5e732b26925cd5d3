# round profile r02m at HEAD: GPU suite (with full-view reports), smoke, bench, launch list, ncu full
mkdir -p gpurun_out/r02m_parity
python -m paper_2411_16392_b200.build > /dev/null 2>&1
QGS_PARITY_OUT=gpurun_out/r02m_parity timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r02m_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/r02m_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
bash tools/round_profile.sh r02m
