# pipelined step, scan first then the estimate beside the slide (bench.py now) vs round 1's order
for C in caida 10G; do for O in scan-first estimate-first; do
  E=staged; [ $C = 10G ] && E=sorted
  python tools/pipe_probe.py --config $C --order $O --estimate $E
done; done
timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 30 --warmup 5 > gpurun_out/b_po_caida.json 2>/dev/null; echo b=$?
timeout 600 python bench.py --config 10G --no-e2e --no-cpu-baseline --steps 20 --warmup 5 > gpurun_out/b_po_10G.json 2>/dev/null; echo b10=$?
for f in caida 10G; do python -c "import json; d=json.load(open('gpurun_out/b_po_$f.json')); c=d['config']; print('$f step',d['ms_per_step'],'serial',d['ms_per_step_serial'],'pipe',c['ms_per_step_pipelined'],c['schedule'][:9])"; done
