# ncu --set full of the caida scan (layout F, mode 5) and the 10G scan, with source
A="--estimate staged --pipeline off --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_scan" -s 4 -c 1 -o gpurun_out/prof_scan_caida python bench.py $A > gpurun_out/ncu_scan_caida.log 2>&1; echo ncu_c=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_scan" -s 4 -c 1 -o gpurun_out/prof_scan_10G python bench.py --config 10G --estimate sorted --pipeline off --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_scan_10G.log 2>&1; echo ncu_10=$?
