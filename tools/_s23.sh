mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py -m gpu -x -q > gpurun_out/r2s_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2s_tests.log
H2B_SETUP_VERBOSE=1 timeout 300 python tools/setup_only.py 1048576 2 > gpurun_out/r2s_setup.log 2>&1
for c in c1 c3; do timeout 600 python tools/setup_cfg.py $c 2 > gpurun_out/r2s_setup_$c.log 2>&1; done
