# C register ranges on the round-2 kernel (per-warp finish, log table): parity, A/B, trace
for C in 2; do VBDR_PLAN_RANGES=$C timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -k "plan or random_config" -q -x > gpurun_out/pytest_r$C.log 2>&1; echo pytest_r$C=$?; tail -1 gpurun_out/pytest_r$C.log; done
A="--estimate staged --no-e2e --no-cpu-baseline --steps 30 --warmup 5"
for C in 1 2 4; do VBDR_PLAN_RANGES=$C TAG=r$C bash tools/ab.sh "$A" main; done
cp tools/var_build/trace/libvbdr.so paper_1810_13132_b200/_lib/libvbdr.so
for C in 2 4; do echo "C=$C"; VBDR_PLAN_RANGES=$C python tools/plan_trace.py 2>&1 | tail -6; done
