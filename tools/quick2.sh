mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py -x -q -k "${PYTEST_K:-m2l or full_size or let}" 2>&1 | tail -2
for c in ${CONFIGS:-c2 c3 c4}; do
python bench.py --no-cpu-baseline --no-probe --steps 5 --config $c 2>gpurun_out/q2_err.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['roofline']['stages_ms'].items()})"
done
