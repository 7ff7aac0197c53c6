# One measurement pass on a B200 (run under gpurun from the repo root).
# At most one ncu per gpurun call: this script takes the launch list; the
# full capture is tools/gpu_ncu_full.sh (a separate call).
set -u
nproc > gpurun_out/nproc.txt; lscpu | grep -E "Model name|^CPU\(s\)" >> gpurun_out/nproc.txt
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python bench.py > gpurun_out/bench_caida_fast.json 2> gpurun_out/bench_caida_fast.err; echo bench=$?
timeout 300 python bench.py --layout packed --no-cpu-baseline > gpurun_out/bench_caida_packed.json 2> gpurun_out/bench_caida_packed.err; echo bench_packed=$?
timeout 600 python bench.py --config 10G --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/bench_10G_fast.json 2> gpurun_out/bench_10G.err; echo bench_10G=$?
timeout 600 python bench.py --config bigwin --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/bench_bigwin_fast.json 2> gpurun_out/bench_bigwin.err; echo bench_bigwin=$?
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err; echo bench_ref=$?
ARGS="--steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 300 python bench.py $ARGS > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py $ARGS > gpurun_out/ncu_launches.log 2>&1; echo ncu1=$?
