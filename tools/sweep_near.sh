
mkdir -p gpurun_out
b() { python bench.py --no-cpu-baseline --no-probe --steps 5 "$@" 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$TAG', round(d['ms_per_step'],3), 'near', round(d['roofline']['stages_ms']['near'],3))"; }
TAG="default" b
TAG="default c2 grad" b --config c2
for tg in "2 8" "4 4" "4 2" "3 8"; do set -- $tg; TAG="T<=$1 G<=$2" FMM_NEAR_MAXTPL=$1 FMM_NEAR_MAXG=$2 b; done
ncu --set full --clock-control none --import-source on -k regex:near_warp -s 2 -c 1 -o gpurun_out/near3_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-probe > gpurun_out/ncu_near3.log 2>&1
for ex in "-DFMM_NEAR_MINB=3" "-DFMM_NEAR_UNROLL=1" "-DFMM_NEAR_UNROLL=4"; do
  FMM_NVCC_EXTRA="$ex" python -c "from paper_1602_02244_b200 import build; build.build(force=True)"
  TAG="$ex" b
done
