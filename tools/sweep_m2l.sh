mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py -x -q -k "m2l or expansions" 2>&1 | tail -1
b() { python bench.py --no-cpu-baseline --no-probe --steps 5 "$@" 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$TAG', round(d['ms_per_step'],3), 'm2l', round(d['roofline']['stages_ms']['m2l'],3))"; }
for d in 0 14; do TAG="mma12 dbg=$d" FMM_M2L_DEBUG=$d b; done
for M in 8 16; do
FMM_NVCC_EXTRA=-DFMM_ROT_MMA=$M python -c "from paper_1602_02244_b200 import build; build.build(force=True)" > /dev/null 2>&1
for d in 0 14; do TAG="mma$M dbg=$d" FMM_M2L_DEBUG=$d b; done
done
