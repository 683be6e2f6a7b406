# M2L v3 timing ablations (FMM_M2L_DEBUG bits skip work: results are wrong, timing only)
# 2 prep compute, 4 accumulate, 16 stage barriers, 32 MMA stores, 64 MMA B loads, 1 all MMA items
mkdir -p gpurun_out
for d in ${DBGS:-0 64 32 96 16 112 6 1 7}; do
FMM_M2L_DEBUG=$d python bench.py --no-cpu-baseline --no-probe --steps 3 --config c3 2>gpurun_out/abl_err.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('dbg $d m2l', round(d['roofline']['stages_ms']['m2l'],3))"
done
