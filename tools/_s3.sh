mkdir -p gpurun_out
H2B_SETUP_VERBOSE=1 timeout 600 python bench.py --no-cpu-baseline > gpurun_out/t3_bench_c2.json 2> gpurun_out/t3_bench_c2.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/t3_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/t3_ncu_launch.log 2>&1
