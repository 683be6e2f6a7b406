mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py -x -q -k "near or edge or expansions or full_size" > gpurun_out/exp_pytest.log 2>&1; tail -3 gpurun_out/exp_pytest.log
python bench.py --no-cpu-baseline --no-probe > gpurun_out/exp_b3.log 2>&1; tail -1 gpurun_out/exp_b3.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('minb3', d['ms_per_step'], d['roofline']['stages_ms'])"
python bench.py --no-cpu-baseline --no-probe --config c2 > gpurun_out/exp_b3c2.log 2>&1; tail -1 gpurun_out/exp_b3c2.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('minb3 c2', d['ms_per_step'], d['roofline']['stages_ms'])"
FMM_NVCC_EXTRA=-DFMM_NEAR_MINB=4 python -c "from paper_1602_02244_b200 import build; build.build(force=True)"
python bench.py --no-cpu-baseline --no-probe > gpurun_out/exp_b4.log 2>&1; tail -1 gpurun_out/exp_b4.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('minb4', d['ms_per_step'], d['roofline']['stages_ms'])"
python bench.py --no-cpu-baseline --no-probe --config c2 > gpurun_out/exp_b4c2.log 2>&1; tail -1 gpurun_out/exp_b4c2.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('minb4 c2', d['ms_per_step'], d['roofline']['stages_ms'])"
