# A/B of M2M/L2L variants + parity subset
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py -x -q -k "expansions or edge or full_size or matvec" > gpurun_out/s_pytest.log 2>&1; tail -3 gpurun_out/s_pytest.log
for c in ${CONFIGS:-c3 c4 c5}; do
for v in ${VARIANTS:-"FMM_SHIFT_VARIANT=1" "FMM_SHIFT_PAR=2" "FMM_SHIFT_PAR=1"}; do
env $v python bench.py --no-cpu-baseline --no-probe --steps 5 --config $c 2>gpurun_out/s_bench_err.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c $v', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['roofline']['stages_ms'].items()})"
done
done
