# staged plan with smaller register blocks (smaller stages): room on the SM for the scan and
# slide of the next slice in the pipelined schedule (caida)
A="--estimate staged --no-e2e --no-cpu-baseline --steps 30 --warmup 5"
for BL in 16 15 14 13; do
  VBDR_PLAN_BLOCK_LOG2=$BL timeout 300 python bench.py $A > gpurun_out/b_bl$BL.json 2> gpurun_out/b_bl$BL.err; echo bl$BL=$?
  python -c "import json; d=json.load(open('gpurun_out/b_bl$BL.json')); c=d['config']; print('bl $BL step',d['ms_per_step'],'serial',d['ms_per_step_serial'],'pipelined',c.get('ms_per_step_pipelined'),'scan',d['scan_mpairs_s'],'slide',d['slide_ms'],'est',d['estimate_ms'])"
done
timeout 900 python -m pytest tests/test_gpu_parity.py -k "plan" -q -x > gpurun_out/pytest_plan3.log 2>&1; echo pytest_plan=$?; tail -2 gpurun_out/pytest_plan3.log
