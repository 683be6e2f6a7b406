# One GPU session's evidence (run under gpurun from the repo root): tests, smoke, benches,
# the ncu launch list and full captures of the two top kernels. Outputs in gpurun_out/.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "from oracle import oracle as O; O.build()"
python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
python bench.py > gpurun_out/bench.log 2>&1
python bench.py --config c2 --no-cpu-baseline > gpurun_out/bench_c2.log 2>&1
python bench.py --config c4 --no-cpu-baseline --steps 5 > gpurun_out/bench_c4.log 2>&1
python bench.py --config c5 --no-cpu-baseline --steps 3 > gpurun_out/bench_c5.log 2>&1
python bench.py --config l3 --no-cpu-baseline --steps 5 > gpurun_out/bench_l3.log 2>&1
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-probe > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-probe > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:m2l_v4_kernel -s 1 -c 1 -o gpurun_out/m2l_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-probe > gpurun_out/ncu_m2l.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:near_mutual_kernel -s 1 -c 1 -o gpurun_out/near_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-probe > gpurun_out/ncu_near.log 2>&1
for f in gpurun_out/*.log; do echo "== $f"; tail -n 3 $f; done
