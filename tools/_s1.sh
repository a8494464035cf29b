bash tools/gpu_session.sh r2b
timeout 900 ncu --set full --clock-control none --import-source on -k regex:interact_sym -s 3 -c 1 -o gpurun_out/r2b_interact_sym python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r2b_ncu_full.log 2>&1
