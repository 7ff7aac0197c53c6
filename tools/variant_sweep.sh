# usage: bash tools/variant_sweep.sh v1 v2 ...   (tools/variants/<v>/libvbdr.so)
OUT=gpurun_out/variants.txt
: > $OUT
for rep in 1 2; do
for v in "$@"; do
  for cfg in "caida fast" "caida packed" "10G fast"; do
    set -- $cfg
    steps=200; [ "$1" = "10G" ] && steps=20
    VBDR_LIB=tools/variants/$v/libvbdr.so timeout 300 python bench.py --config $1 --layout $2 --steps $steps --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/v.json 2>/dev/null
    python - "$v" "$1" "$2" >> $OUT <<'PY'
import json,sys
d=json.loads(open("gpurun_out/v.json").read().strip().splitlines()[-1]); k=d["kernels"]
print(f"{sys.argv[1]:10s} {sys.argv[2]:6s} {sys.argv[3]:6s} step={d['ms_per_step']*1e3:8.1f}us scan={k['scan']['ms']*1e3:7.1f} slide={k['slide']['ms']*1e3:7.1f} ({k['slide']['frac']:.3f}) est={k['estimate']['ms']*1e3:7.1f}")
PY
  done
done
done
cat $OUT
