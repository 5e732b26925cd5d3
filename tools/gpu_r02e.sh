# full GPU suite with parity reports (tag r02e)
mkdir -p gpurun_out
QGS_PARITY_OUT=gpurun_out/r02e_parity timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r02e_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r02e_tests.log
