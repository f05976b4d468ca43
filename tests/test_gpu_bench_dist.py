"""GPU: bench.py's N>1 cooperative arm (one part per rank, exchange through
torch.distributed) end to end at world size 2. The pool gives one GPU per
call, so both ranks share cuda:0 over gloo (--dist-backend gloo); on a
multi-GPU node the same code runs over NCCL."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_coop_world2(gpu):
    from tests.dist_harness import free_port
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", "bench.py", "--gpus", "2",
           "--steps", "4", "--warmup", "3", "--config", "c1", "--dist-backend", "gloo"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["e2e"]["value"] > 0
    assert d["gpu_launches"] > 0 and "cooperative" in d["config"]["mode"]
