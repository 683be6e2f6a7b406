mkdir -p gpurun_out
for lib in libfmm.so libfmm_nc16.so libfmm_nc40.so libfmm_nc64.so; do for d in 0 6; do
FMM_LIB=$lib FMM_M2L_DEBUG=$d python bench.py --no-cpu-baseline --no-probe --steps 3 --config c3 2>gpurun_out/nc_err.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib dbg $d m2l', round(d['roofline']['stages_ms']['m2l'],3))"
done; done
FMM_LIB=libfmm_nc64.so python -m pytest tests/test_gpu_parity.py -q -x -k "m2l_variants" 2>&1 | tail -1
