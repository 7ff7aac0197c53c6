# ncu --set full of the staged-plan estimate with 1 and 4 register ranges (caida)
A="--estimate staged --pipeline off --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
for C in 1 4; do
  VBDR_PLAN_RANGES=$C timeout 300 python bench.py $A > gpurun_out/plain_r$C.log 2>&1 && \
  VBDR_PLAN_RANGES=$C timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_estimate_plan" -s 6 -c 1 -o gpurun_out/prof_plan_r$C python bench.py $A > gpurun_out/ncu_plan_r$C.log 2>&1; echo ncu_r$C=$?
done
