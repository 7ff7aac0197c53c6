# NCCL group-of-one merges + the gloo multi-rank tests (worker changed)
timeout 900 python -m pytest tests/test_gpu_dist.py -q > gpurun_out/pytest_dist.log 2>&1; echo pytest_dist=$?; tail -15 gpurun_out/pytest_dist.log
