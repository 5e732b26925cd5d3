# shared-reciprocal key division: debug-build equality checks at full C3 / C4 views, sort tests, A/B
python -m paper_2411_16392_b200.build > /dev/null 2>&1
for c in c3 c4; do QGS_LIB_VARIANT=debug timeout 900 python tools/sanitize_view.py --config $c > /tmp/san_$c.log 2>&1; echo "debug $c rc=$?"; grep -c "QGS_CHECK failed" /tmp/san_$c.log; tail -1 /tmp/san_$c.log; done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_debug_checks.py -q -k "binning or sort or debug" 2>&1 | tail -1
CFGS="c3 c4" bash tools/gpu_exp_cfg.sh "" "-DQGS_KEY_SHARED_RCP=0"
