# ncu --set full of the 10G step's kernels (layout F, sorted-plan estimate)
A="--config 10G --estimate sorted --pipeline off --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_scan|k_slide|k_estimate" -s 9 -c 3 -o gpurun_out/prof_final_10G python bench.py $A > gpurun_out/ncu_full_10G.log 2>&1; echo ncu=$?
