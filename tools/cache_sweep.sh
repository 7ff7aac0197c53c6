OUT=gpurun_out/cache.txt
: > $OUT
for v in c1024 c2048 c4096; do
for cfg in caida:200 10G:20; do
  c=${cfg%%:*}; steps=${cfg##*:}
  VBDR_LIB=tools/variants/$v/libvbdr.so timeout 300 python bench.py --config $c --steps $steps --warmup 3 --no-e2e --no-cpu-baseline --scan-mode 5 > gpurun_out/m.json 2>gpurun_out/m.err
  python - "$v" "$c" >> $OUT <<'PY'
import json,sys
d=json.loads(open("gpurun_out/m.json").read().strip().splitlines()[-1]); k=d["kernels"]
print(f"{sys.argv[1]} {sys.argv[2]:6s} scan={k['scan']['ms']*1e3:8.1f}us")
PY
done; done
cat $OUT
