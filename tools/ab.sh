# A/B of compile-time variants of libfmm.so on the GPU box (measurement only).
#   here:    tools/ab.sh build NAME "-DKNOB=1 ..."     (builds ab_libs/NAME/libfmm.so with those flags)
#   on GPU:  tools/ab.sh run "c3 c4" NAME1 NAME2 ...   (installs each and prints its bench stage times)
# ab_libs/ is git-ignored but travels with gpurun. The default build is restored afterwards.
set -e
cmd=$1; shift
LIBDIR=paper_1602_02244_b200
if [ "$cmd" = build ]; then
  name=$1; flags=$2
  mkdir -p ab_libs/$name
  FMM_NVCC_EXTRA="$flags" python -c "from paper_1602_02244_b200 import build as B; B.BUILD = B.BUILD + '_ab'; B.build(force=True)"
  cp $LIBDIR/libfmm.so ab_libs/$name/libfmm.so
  cp $LIBDIR/libfmm.so.flags ab_libs/$name/libfmm.so.flags
  echo "$flags" > ab_libs/$name/FLAGS
  [ -n "$AB_NO_RESTORE" ] || python -c "from paper_1602_02244_b200 import build as B; B.build(force=True)"
elif [ "$cmd" = run ]; then
  cfgs=$1; shift
  cp $LIBDIR/libfmm.so /tmp/libfmm.default.so; cp $LIBDIR/libfmm.so.flags /tmp/libfmm.default.flags
  for name in "$@"; do
    for c in $cfgs; do
      cp ab_libs/$name/libfmm.so $LIBDIR/libfmm.so; cp ab_libs/$name/libfmm.so.flags $LIBDIR/libfmm.so.flags
      touch $LIBDIR/libfmm.so
      steps=10; [ $c = c5 ] && steps=3
      FMM_NVCC_EXTRA="$(cat ab_libs/$name/FLAGS)" python bench.py --config $c --no-cpu-baseline --no-probe --steps $steps 2>/dev/null | tail -1 | \
        python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$name', '$c', round(d['ms_per_step'],3), {k: round(v,3) for k,v in r['stages_ms'].items()}, 'frac', round(r['frac'],3), 'p2p_m2l', round(r['p2p_m2l_frac'],3))"
    done
  done
  cp /tmp/libfmm.default.so $LIBDIR/libfmm.so; cp /tmp/libfmm.default.flags $LIBDIR/libfmm.so.flags; touch $LIBDIR/libfmm.so
fi
