mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/t2_tests.log 2>&1; echo "rc=$?" >> gpurun_out/t2_tests.log
H2B_SETUP_VERBOSE=1 timeout 600 python bench.py --no-cpu-baseline > gpurun_out/t2_bench_c2.json 2> gpurun_out/t2_bench_c2.err
timeout 900 python bench.py --config c4 --steps 5 --no-cpu-baseline > gpurun_out/t2_bench_c4.json 2> gpurun_out/t2_bench_c4.err
