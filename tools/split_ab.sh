mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py -x -q -k "split" 2>&1 | tail -3
for c in c2 c3; do for s in 1 2 4; do
FMM_M2L_SPLIT=$s python bench.py --no-cpu-baseline --no-probe --steps 5 --config $c 2>gpurun_out/split_err.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c split $s', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['roofline']['stages_ms'].items()})"
done; done
tail -3 gpurun_out/split_err.log
