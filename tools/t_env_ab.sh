mkdir -p gpurun_out
for c in ${CONFIGS:-c5}; do for t in ${TS:-default 32}; do
if [ "$t" = "default" ]; then unset FMM_M2L_T; else export FMM_M2L_T=$t; fi
python bench.py --no-cpu-baseline --no-probe --steps 3 --config $c 2>gpurun_out/t_err.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c T=$t', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['roofline']['stages_ms'].items()})"
done; done
unset FMM_M2L_T
