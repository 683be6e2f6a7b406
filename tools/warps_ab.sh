mkdir -p gpurun_out
for lib in libfmm.so libfmm_m12a4.so libfmm_m10a6.so libfmm_m16a4.so; do
FMM_LIB=$lib python bench.py --no-cpu-baseline --no-probe --steps 5 --config c3 2>gpurun_out/w_err.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['roofline']['stages_ms'].items()})"
done
