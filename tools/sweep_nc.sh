b() { python bench.py --no-cpu-baseline --no-probe --steps 3 --config $1 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(\"$TAG $1\", round(d[\"ms_per_step\"],3), {k: round(v,3) for k,v in d[\"roofline\"][\"stages_ms\"].items()})"; }
for nc in 64 48 56; do
FMM_NVCC_EXTRA=-DFMM_ROT_NC=$nc python -c "from paper_1602_02244_b200 import build; build.build(force=True)" > /dev/null 2>&1
TAG="nc$nc" b c3; TAG="nc$nc" b c4
done
