# A/B of libvbdr.so builds on one GPU box (run under gpurun from the repo root).
# usage: TAG=x bash tools/ab.sh "<bench args>" main variant1 variant2 ...
#   main = the in-tree build; others = tools/var_build/<name>/libvbdr.so
#   (tools/build_variant.py).  Bench lines go to gpurun_out/ab_<TAG>_<name>.json.
set -u
TAG=${TAG:-x}
ARGS=$1; shift
LIB=paper_1810_13132_b200/_lib/libvbdr.so
cp $LIB /tmp/ab_main.so
for v in "$@"; do
  if [ "$v" = main ]; then cp /tmp/ab_main.so $LIB; else cp tools/var_build/$v/libvbdr.so $LIB; fi
  O=gpurun_out/ab_${TAG}_$v
  timeout 300 python bench.py $ARGS > $O.json 2> $O.err
  echo "$TAG $v rc=$? $(python -c "import json,sys; d=json.load(open('$O.json')); print('step',d['ms_per_step'],'serial',d.get('ms_per_step_serial'),'scan',d['scan_mpairs_s'],'slide',d['slide_ms'],'est',d['estimate_ms'],d['config']['estimate_autotune'])" 2>&1 | tail -1)"
done
cp /tmp/ab_main.so $LIB
