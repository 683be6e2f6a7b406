mkdir -p gpurun_out
for c in ${CONFIGS:-c3 c4 c5}; do for v in ${VARIANTS:-"X=0"}; do
env $v python bench.py --no-cpu-baseline --no-probe --steps 3 --config $c 2>gpurun_out/ne_err.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c $v', round(d['ms_per_step'],3), 'near', round(d['roofline']['stages_ms']['near'],3))"
done; done
