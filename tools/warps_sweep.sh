# M2L v4 time at 3..7 warps per SM (FMM_V4_WARPS) at configs[2], [4], [3]: run under gpurun from the repo root
# (profiles/r2_m2l_bound.md quotes the result).
for w in 3 4 5 6 7; do
FMM_V4_WARPS=$w python bench.py --config c3 --no-cpu-baseline --no-probe --steps 10 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3 warps $w', round(d['ms_per_step'],3), d['roofline']['stages_ms']['m2l'])"
done
for w in 2 3 4 5; do
FMM_V4_WARPS=$w python bench.py --config c5 --no-cpu-baseline --no-probe --steps 3 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c5 warps $w', round(d['ms_per_step'],3), d['roofline']['stages_ms']['m2l'])"
done
for w in 4 6 8; do
FMM_V4_WARPS=$w python bench.py --config c4 --no-cpu-baseline --no-probe --steps 5 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c4 warps $w', round(d['ms_per_step'],3), d['roofline']['stages_ms']['m2l'])"
done
