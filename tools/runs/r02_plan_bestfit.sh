# best-fit round scheduler (caida, staged): bench + ncu + plan parity
A="--estimate staged --no-e2e --no-cpu-baseline --steps 30 --warmup 5"
timeout 300 python bench.py $A > gpurun_out/b_bf.json 2> gpurun_out/b_bf.err; echo bf=$?
python -c "import json; d=json.load(open('gpurun_out/b_bf.json')); c=d['config']; print('step',d['ms_per_step'],'serial',d['ms_per_step_serial'],'est',d['estimate_ms'],'build',c['plan_build_ms'])"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_estimate_plan" -s 6 -c 1 -o gpurun_out/prof_plan_bf python bench.py --estimate staged --pipeline off --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_plan_bf.log 2>&1; echo ncu=$?
timeout 900 python -m pytest tests/test_gpu_parity.py -k "plan" -q -x > gpurun_out/pytest_plan6.log 2>&1; echo pytest_plan=$?; tail -2 gpurun_out/pytest_plan6.log
