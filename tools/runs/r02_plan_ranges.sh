set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -k "plan or e2e_pipelined" -q -x > gpurun_out/pytest_plan.log 2>&1; echo pytest=$?; tail -5 gpurun_out/pytest_plan.log
for C in 1 2 4; do VBDR_PLAN_RANGES=$C timeout 300 python bench.py --estimate staged --no-e2e --no-cpu-baseline --steps 20 --warmup 5 > gpurun_out/b_c$C.json 2> gpurun_out/b_c$C.err; echo c$C=$?; python -c "import json; d=json.load(open('gpurun_out/b_c$C.json')); print('step',d['ms_per_step'],'serial',d['ms_per_step_serial'],'est',d['estimate_ms'])"; done
