# two-byte (accumulator index, i) entries, Alg.3 recomputed in the consumer (caida, staged)
timeout 900 python -m pytest tests/test_gpu_parity.py -k "plan or e2e_pipelined or query_top" -q -x > gpurun_out/pytest_plan7.log 2>&1; echo pytest_plan=$?; tail -3 gpurun_out/pytest_plan7.log
A="--estimate staged --no-e2e --no-cpu-baseline --steps 30 --warmup 5"
timeout 300 python bench.py $A > gpurun_out/b_hash.json 2> gpurun_out/b_hash.err; echo bench=$?
python -c "import json; d=json.load(open('gpurun_out/b_hash.json')); c=d['config']; print('step',d['ms_per_step'],'serial',d['ms_per_step_serial'],'est',d['estimate_ms'],'build',c['plan_build_ms'])"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_estimate_plan" -s 6 -c 1 -o gpurun_out/prof_plan_hash python bench.py --estimate staged --pipeline off --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_plan_hash.log 2>&1; echo ncu=$?
