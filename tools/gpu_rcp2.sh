# shared-reciprocal corner projection in tight_box: debug-build equality checks at full C3 / C4 views, parity tests, A/B
python -m paper_2411_16392_b200.build > /dev/null 2>&1
for c in c3 c4 c5; do QGS_LIB_VARIANT=debug timeout 900 python tools/sanitize_view.py --config $c > /tmp/san_$c.log 2>&1; echo "debug $c rc=$?"; grep -c "QGS_CHECK failed" /tmp/san_$c.log; tail -1 /tmp/san_$c.log | cut -c1-80; done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_debug_checks.py tests/test_gpu_known_answers.py tests/test_dist.py -q -m gpu 2>&1 | tail -1
bash tools/gpu_ab.sh preprocess.cu tools/ab/preprocess_old.cu 2>&1 | sed "s/raster_[a-z_]*kernel[^,]*,//g"; ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:chain python tools/profile_view.py --config c3 2>/dev/null | grep -i chain | tail -1 | cut -c1-300
