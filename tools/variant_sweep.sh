# usage: bash tools/variant_sweep.sh v1 v2 ...   (tools/variants/<v>/libvbdr.so)
OUT=gpurun_out/variants.txt
: > $OUT
VARIANTS="$*"
for rep in 1 2; do
for v in $VARIANTS; do
  for cfg in caida:fast caida:packed 10G:fast; do
    c=${cfg%%:*}; lay=${cfg##*:}
    steps=200; [ "$c" = "10G" ] && steps=20
    VBDR_LIB=tools/variants/$v/libvbdr.so timeout 300 python bench.py --config $c --layout $lay --steps $steps --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/v.json 2>gpurun_out/v.err
    python - "$v" "$c" "$lay" >> $OUT <<'PY'
import json,sys
try:
    d=json.loads(open("gpurun_out/v.json").read().strip().splitlines()[-1]); k=d["kernels"]
    print(f"{sys.argv[1]:10s} {sys.argv[2]:6s} {sys.argv[3]:6s} step={d['ms_per_step']*1e3:8.1f}us scan={k['scan']['ms']*1e3:7.1f} slide={k['slide']['ms']*1e3:7.1f} ({k['slide']['frac']:.3f}) est={k['estimate']['ms']*1e3:7.1f}")
except Exception as e:
    print(sys.argv[1:], "FAILED", open("gpurun_out/v.err").read()[-300:])
PY
  done
done
done
cat $OUT
