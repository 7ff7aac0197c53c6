# scan-mode sweep (run under gpurun): caida fast/packed, 10G, bigwin
OUT=gpurun_out/modes.txt
: > $OUT
for cfg in caida:fast caida:packed 10G:fast bigwin:fast; do
  c=${cfg%%:*}; lay=${cfg##*:}
  steps=200; [ "$c" = "10G" ] && steps=20; [ "$c" = "bigwin" ] && steps=10
  for m in 2 5; do
    timeout 300 python bench.py --config $c --layout $lay --steps $steps --warmup 3 --no-e2e --no-cpu-baseline --scan-mode $m > gpurun_out/m.json 2>gpurun_out/m.err
    python - "$m" "$c" "$lay" >> $OUT <<'PY'
import json,sys
try:
    d=json.loads(open("gpurun_out/m.json").read().strip().splitlines()[-1]); k=d["kernels"]
    print(f"mode={sys.argv[1]} {sys.argv[2]:6s} {sys.argv[3]:6s} step={d['ms_per_step']*1e3:9.1f}us scan={k['scan']['ms']*1e3:8.1f}us slide={k['slide']['ms']*1e3:7.1f} est={k['estimate']['ms']*1e3:8.1f}")
except Exception as e:
    print(sys.argv[1:], "FAILED", open("gpurun_out/m.err").read()[-300:])
PY
  done
done
cat $OUT
