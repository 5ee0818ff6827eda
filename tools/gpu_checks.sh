# bounds-checked build (-DRIG_DEBUG_CHECKS, variants/checks.so) over the sanitize driver and the parity tests
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
export RIG_LIB_VARIANT=variants/checks.so
timeout 900 python tools/sanitize_driver.py > gpurun_out/checks_driver.log 2>&1; echo "driver rc=$?"; tail -3 gpurun_out/checks_driver.log
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -q -m gpu -k "not full_configs" > gpurun_out/checks_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/checks_tests.log
