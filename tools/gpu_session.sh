mkdir -p gpurun_out
# usage: bash tools/gpu_session.sh TAG  (runs the GPU suite, the c2 + c4 bench lines and a launch list)
TAG=${1:-r2}
set -x
timeout 1500 python -m pytest tests -m gpu -x -q -s --durations=10 > gpurun_out/${TAG}_gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/${TAG}_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/${TAG}_bench_c2.json 2> gpurun_out/${TAG}_bench_c2.err
timeout 900 python bench.py --config c4 --steps 5 --no-cpu-baseline > gpurun_out/${TAG}_bench_c4.json 2> gpurun_out/${TAG}_bench_c4.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_ncu_launch.log 2>&1
ls -la gpurun_out
