mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py -m gpu -x -q > gpurun_out/r2l_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2l_tests.log
timeout 600 python bench.py --no-cpu-baseline --no-other-configs > gpurun_out/r2l_bench.json 2> gpurun_out/r2l_bench.err
