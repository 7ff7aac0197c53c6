"""Multi-rank runs of the real GPU path on ONE GPU: torchrun with the gloo
backend (CPU collectives, no cross-rank GPU waiting), every merge of
slide_merged, and bench.py's N>1 control flow."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _torchrun(n, *args, env=None):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", f"--master-port={_port()}", *args]
    return subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600,
                          env={**os.environ, **(env or {})})


@pytest.mark.parametrize("mode", ["stamps", "delta", "sharded", "sparse", "sharded-state"])
@pytest.mark.parametrize("world", [2, 4])
def test_slide_merged_multi_rank(mode, world):
    r = _torchrun(world, os.path.join("tests", "dist_worker.py"), mode)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert f"parity=ok" in r.stdout


@pytest.mark.parametrize("mode", ["stamps", "delta", "sharded", "sparse", "sharded-state", "p2p"])
def test_slide_merged_nccl_group_of_one(mode):
    """Every merge through the NCCL backend (all_reduce MAX on u32 / u8,
    reduce_scatter_tensor MAX, all_gather_into_tensor, all_to_all_single, SUM
    of the pool sums) and PeerMerge's symmetric-memory rendezvous and device
    barriers, on the device tensors, with a group of one: oracle parity at
    every boundary.  (One GPU per box: more NCCL ranks need more GPUs.)"""
    r = _torchrun(1, os.path.join("tests", "dist_worker.py"), mode,
                  env={"VBDR_TEST_BACKEND": "nccl"})
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert "parity=ok" in r.stdout


@pytest.mark.parametrize("merge", ["sharded", "sparse"])
def test_bench_two_ranks_gloo_same_device(merge):
    r = _torchrun(2, "bench.py", "--gpus", "2", "--steps", "5", "--warmup", "3", "--config", "tiny",
                  "--dist-backend", "gloo", "--same-device", "--no-cpu-baseline", "--merge", merge)
    assert r.returncode == 0, r.stderr[-4000:]
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["value"] > 0 and line["gpu_launches"] > 0
    assert f"merge={merge}" in line["config"]["parallelism"]
    assert "communicator of 2 ranks" in r.stderr


@pytest.mark.parametrize("layout", ["fast", "packed"])
def test_bench_one_gpu_multicast_slide(layout):
    """bench.py --merge nvls on one GPU: the NVLS merge + slide kernel through a
    one-device multicast object inside the timed steps."""
    r = subprocess.run([sys.executable, "bench.py", "--steps", "4", "--warmup", "3", "--config",
                        "tiny", "--merge", "nvls", "--layout", layout, "--no-cpu-baseline"],
                       cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-4000:]
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert "multicast" in line["config"]["parallelism"] and line["value"] > 0
