# does a scan without shared memory (mode 2) co-run with the staged estimate in the pipelined step?
A="--estimate staged --no-e2e --no-cpu-baseline --steps 30 --warmup 5"
for M in 5 2; do timeout 300 python bench.py $A --scan-mode $M > gpurun_out/b_m$M.json 2>/dev/null; python -c "import json; d=json.load(open('gpurun_out/b_m$M.json')); c=d['config']; print('mode $M step',d['ms_per_step'],'serial',d['ms_per_step_serial'],'pipe',c['ms_per_step_pipelined'],'scan',d['scan_mpairs_s'],'est',d['estimate_ms'])"; done
timeout 300 nsys --version > /dev/null 2>&1 || echo no-nsys
