# near-field rsqrt refinement order A/B (libfmm.so = order 3, libfmm_o2.so = order 2)
mkdir -p gpurun_out
./tools/rsqrt_probe
FMM_LIB=libfmm_o2.so python -m pytest tests/test_gpu_parity.py -x -q -k "near or edge or full_size" 2>&1 | tail -3
for c in c3 c4; do for lib in libfmm.so libfmm_o2.so; do
FMM_LIB=$lib python bench.py --no-cpu-baseline --no-probe --steps 5 --config $c 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c $lib', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['roofline']['stages_ms'].items()})"
done; done
