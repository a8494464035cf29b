mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/r2g_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2g_tests.log
timeout 600 python tools/setup_variants.py paper_2203_14832_b200/libh2b200.so > gpurun_out/r2g_setup.log 2>&1
