# linear-counting log table + exact 1/g in the plan finishes (caida staged, 10G sorted)
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -k "plan or e2e_pipelined or query_top or random_config or estimator" -q -x > gpurun_out/pytest_lct.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_lct.log
A="--estimate staged --no-e2e --no-cpu-baseline --steps 30 --warmup 5"
TAG=lct bash tools/ab.sh "$A" main main
#TAG=lct10 bash tools/ab.sh "--config 10G --estimate sorted --no-e2e --no-cpu-baseline --steps 10 --warmup 5" main
cp tools/var_build/trace/libvbdr.so paper_1810_13132_b200/_lib/libvbdr.so && python tools/plan_trace.py 2>&1 | tail -6
