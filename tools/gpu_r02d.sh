mkdir -p gpurun_out/r02d
(time QGS_PARITY_OUT=gpurun_out/r02d timeout 900 python -m pytest tests/test_gpu_fullview.py -q -rf -s) > gpurun_out/r02d_tests.log 2>&1; echo "tests rc=$?"
tail -5 gpurun_out/r02d_tests.log
