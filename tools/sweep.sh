# kernel-variant sweep on caida (run under gpurun); one JSON line per variant
set -u
OUT=gpurun_out/sweep.jsonl
: > $OUT
for sm in 1 2 4; do
  for el in 1 2 4 8 32; do
    timeout 120 python bench.py --steps 100 --warmup 5 --no-e2e --no-cpu-baseline --scan-mode $sm --est-lanes $el >> $OUT 2>> gpurun_out/sweep.err || echo "fail sm=$sm el=$el" >> gpurun_out/sweep.err
  done
done
for lay in packed; do
  for sm in 1 2 4; do
    timeout 120 python bench.py --steps 100 --warmup 5 --no-e2e --no-cpu-baseline --layout $lay --scan-mode $sm >> $OUT 2>> gpurun_out/sweep.err
  done
done
python - <<'PY'
import json
for l in open("gpurun_out/sweep.jsonl"):
    d=json.loads(l); c=d["config"]
    print(f'{c["layout"]:6s} scan_mode={c["scan_mode"]} lanes={c["est_lanes"]:2d}  step={d["ms_per_step"]:.4f}ms value={d["value"]:9.1f}  scan={d["kernels"]["scan"]["ms"]*1e3:6.1f}us slide={d["kernels"]["slide"]["ms"]*1e3:6.1f}us ({d["kernels"]["slide"]["frac"]:.3f}) est={d["kernels"]["estimate"]["ms"]*1e3:6.1f}us')
PY
