mkdir -p gpurun_out
for D in ${DBGS:-11}; do
FMM_M2L_DEBUG=$D ncu --set full --clock-control none --import-source on -k regex:m2l_rot -s 1 -c 1 -o gpurun_out/m2l3_full$D python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-probe > gpurun_out/ncu_m2l3.log 2>&1
done
