mkdir -p gpurun_out
timeout 1700 python -m pytest tests -m gpu -x -q --durations=4 > gpurun_out/r2k_gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2k_gpu_tests.log
H2B_SETUP_VERBOSE=1 timeout 900 python bench.py > gpurun_out/r2k_bench_line.json 2> gpurun_out/r2k_bench.err; echo "bench rc=$?" >> gpurun_out/r2k_bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2k_bench_line_reference_arm.json 2> gpurun_out/r2k_bench_ref.err
