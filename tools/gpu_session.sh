mkdir -p gpurun_out
# usage: bash tools/gpu_session.sh TAG [aca]  (GPU suite, smoke, the default bench line + reference arm, a launch list of the
# bench, and ncu --set full captures of the interaction kernel and of the two largest ACA launches)
TAG=${1:-r2}
timeout 1700 python -m pytest tests -m gpu -x -q --durations=8 > gpurun_out/${TAG}_gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/${TAG}_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
H2B_SETUP_VERBOSE=1 timeout 900 python bench.py > gpurun_out/${TAG}_bench_line.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?" >> gpurun_out/${TAG}_bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${TAG}_bench_line_reference_arm.json 2> gpurun_out/${TAG}_bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-other-configs > gpurun_out/${TAG}_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:interact_sym -s 3 -c 1 -o gpurun_out/${TAG}_interact_sym python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-other-configs > gpurun_out/${TAG}_ncu_full_sym.log 2>&1
# (gpurun copies back at most 64 MiB: capture the ACA launches in a call of their own)
if [ "$2" = "aca" ]; then timeout 900 ncu --set full --clock-control none --import-source on -k regex:aca_ring -c 2 -o gpurun_out/${TAG}_aca_ring python tools/setup_only.py 1048576 1 > gpurun_out/${TAG}_ncu_full_aca.log 2>&1; fi
ls -la gpurun_out
