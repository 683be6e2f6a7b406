mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py -x -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/q_pytest.log 2>&1; tail -3 gpurun_out/q_pytest.log
for c in ${CONFIGS:-c3 c2}; do
python bench.py --no-cpu-baseline --no-probe --steps 5 --config $c 2>gpurun_out/q_bench_err.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['roofline']['stages_ms'].items()}, '%.3g p/s' % d['value'])"
done
