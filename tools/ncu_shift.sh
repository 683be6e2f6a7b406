mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_s.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-probe > gpurun_out/ncu_launch_s.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"shift_dmma|p2m_warp" -c 4 -o gpurun_out/shift_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-probe > gpurun_out/ncu_shift.log 2>&1
tail -2 gpurun_out/ncu_shift.log
