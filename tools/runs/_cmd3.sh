set -u
A="--no-e2e --no-cpu-baseline --steps 20 --warmup 5"
TAG=spc bash tools/ab.sh "$A --estimate sorted" main sp_u16pf64 sp_u8pf128 sp_u8pf32
TAG=sp10 bash tools/ab.sh "$A --estimate sorted --config 10G" main sp_u16pf64 sp_u8pf128 sp_u8pf32
B="--no-e2e --no-cpu-baseline --steps 3 --warmup 3 --pipeline off"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_estimate_sp|k_scan" -s 2 -c 2 -o gpurun_out/prof_sp_caida python bench.py $B --estimate sorted > gpurun_out/ncu_sp_caida.log 2>&1; echo ncu_c=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_estimate_sp|k_scan" -s 2 -c 2 -o gpurun_out/prof_sp_10G python bench.py $B --estimate sorted --config 10G > gpurun_out/ncu_sp_10G.log 2>&1; echo ncu_10=$?
