mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py -m gpu -x -q > gpurun_out/r2m_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2m_tests.log
H2B_SETUP_VERBOSE=1 timeout 300 python tools/setup_only.py 1048576 2 > gpurun_out/r2m_setup.log 2>&1
