mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py -x -q -k "m2l or expansions" 2>&1 | tail -1
b() { python bench.py --no-cpu-baseline --no-probe --steps 5 "$@" 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$TAG', round(d['ms_per_step'],3), 'm2l', round(d['roofline']['stages_ms']['m2l'],3))"; }
for d in 0 1 14 13 11 7; do TAG="dbg=$d" FMM_M2L_DEBUG=$d b; done
