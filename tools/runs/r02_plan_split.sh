# 3-byte entries in two planes (u16 offsets + u8 accumulator indices), caida staged
timeout 900 python -m pytest tests/test_gpu_parity.py -k "plan or e2e_pipelined or query_top" -q -x > gpurun_out/pytest_plan8.log 2>&1; echo pytest_plan=$?; tail -3 gpurun_out/pytest_plan8.log
A="--estimate staged --no-e2e --no-cpu-baseline --steps 30 --warmup 5"
TAG=sp bash tools/ab.sh "$A" main
VBDR_PLAN_SPLIT=0 TAG=u32 bash tools/ab.sh "$A" main
TAG=sp2 bash tools/ab.sh "$A" main
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_estimate_plan" -s 6 -c 1 -o gpurun_out/prof_plan_split python bench.py --estimate staged --pipeline off --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_plan_split.log 2>&1; echo ncu=$?
