set -u
A="--no-e2e --no-cpu-baseline --steps 20 --warmup 5"
TAG=spc bash tools/ab.sh "$A --estimate sorted" main sp_u16 sp_pf0 sp_pf32
TAG=sp10 bash tools/ab.sh "$A --estimate sorted --config 10G" main sp_u16 sp_pf0 sp_pf32
B="--no-e2e --no-cpu-baseline --steps 3 --warmup 3 --pipeline off"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_estimate_sp" -s 1 -c 1 -o gpurun_out/prof_sp2_10G python bench.py $B --estimate sorted --config 10G > gpurun_out/ncu_sp2_10G.log 2>&1; echo ncu_10=$?
