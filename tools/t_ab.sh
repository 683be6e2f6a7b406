mkdir -p gpurun_out
for c in ${CONFIGS:-c3 c4}; do for v in "libfmm.so 64" "libfmm_l2a.so 64" "libfmm_l2a.so 128" "libfmm_l2a.so 256"; do set -- $v
FMM_LIB=$1 FMM_M2L_T=$2 python bench.py --no-cpu-baseline --no-probe --steps 5 --config $c 2>gpurun_out/t_err.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c $1 T=$2', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['roofline']['stages_ms'].items()})"
done; done
