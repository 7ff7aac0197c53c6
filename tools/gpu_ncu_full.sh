# ncu --set full of the step's kernels (scan, slide, estimate) at caida;
# usage: bash tools/gpu_ncu_full.sh <fast|packed>
set -u
L=${1:-fast}
ARGS="--steps 3 --warmup 3 --no-e2e --no-cpu-baseline --layout $L"
timeout 300 python bench.py $ARGS > gpurun_out/plain_$L.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_scan|k_slide|k_estimate" -s 9 -c 3 -o gpurun_out/prof_caida_$L python bench.py $ARGS > gpurun_out/ncu_full_$L.log 2>&1; echo ncu=$?
