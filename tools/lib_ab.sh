# A/B of alternative in-tree libraries: LIBS="libfmm.so libfmm_x.so" CONFIGS="c3 c4" bash tools/lib_ab.sh
mkdir -p gpurun_out
if [ -n "$PYTEST_K" ]; then for lib in $LIBS; do FMM_LIB=$lib python -m pytest tests/test_gpu_parity.py -x -q -k "$PYTEST_K" 2>&1 | tail -1; done; fi
for c in ${CONFIGS:-c3}; do for lib in $LIBS; do
FMM_LIB=$lib python bench.py --no-cpu-baseline --no-probe --steps ${STEPS:-5} --config $c 2>gpurun_out/lib_err.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c $lib', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['roofline']['stages_ms'].items()})"
done; done
