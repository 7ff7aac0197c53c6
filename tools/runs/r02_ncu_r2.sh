A="--estimate staged --pipeline off --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
VBDR_PLAN_RANGES=2 timeout 900 ncu --set full --clock-control none -k regex:"k_estimate_plan" -s 6 -c 1 -o gpurun_out/prof_r2 python bench.py $A > gpurun_out/ncu_r2.log 2>&1; echo ncu=$?
