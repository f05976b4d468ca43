"""Programmatic dependent launch on and off (CB_PDL, read once per process)
must produce the same batch: the kernels' griddepcontrol.wait orders them
either way. Each mode runs in its own process."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROG = r"""
import numpy as np, paper_2310_12403_b200 as cb
g = cb.Graph.generate_rmat(1 << 16, 1 << 20, 42)
pm = cb.partition_random(g, 4, 7)
fs = cb.FeatureStore.synth(g, 100, 5, pm=pm)
out = []
for kind in (cb.SamplerKind.kLabor0, cb.SamplerKind.kNs):
    cfg = cb.SamplerConfig(kind, 10)
    pl = cb.Plan(g, pm, 3, cfg, 1024)
    mem = pm.members()
    seeds = [mem[p][:: max(1, len(mem[p]) // 1000)][:1000] for p in range(4)]
    for mode in (cb.MODE_COOP, cb.MODE_INDEP):
        pl.sample(seeds, cb.SeedSchedule.make(1, 3), mode)
        pl.gather(fs)
        for p in range(4):
            out.append(cb.stack_fingerprint(pl, p))
            out.append(int(np.frombuffer(pl.rows(p, fs).tobytes(), np.uint8).astype(np.uint64).sum()))
print(out)
"""


def run(pdl: str) -> str:
    env = dict(os.environ, CB_PDL=pdl)
    r = subprocess.run([sys.executable, "-c", PROG], cwd=ROOT, env=env, capture_output=True,
                       text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    return r.stdout.strip().splitlines()[-1]


def test_pdl_on_off_same_batches(gpu):
    assert run("1") == run("0")
