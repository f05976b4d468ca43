"""Writes tests/golden/c4_csr.json: SHA-256 digests of the config-4 R-MAT CSR
(papers100M-shaped, 111,059,956 V / 1,615,685,872 E, bench.GRAPH_SEED) built
by the oracle's generator (oracle/coopbatch_oracle.c ob_rmat_par, the same
graph as the sequential ob_rmat; tests/test_oracle_golden.py checks the two
agree). The GPU test compares the device CSR against these digests so the
full-size graph need not be regenerated on the CPU at test time.

    python tests/golden/make_c4_digest.py     # ~2 min, ~45 GB host memory
"""
import hashlib
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import bench  # noqa: E402
from oracle import oracle as O  # noqa: E402


def main():
    c = bench.CONFIGS["c4"]
    t0 = time.time()
    g = O.rmat(c["n"], c["m"], bench.GRAPH_SEED)
    deg = np.diff(g.indptr)
    out = {"config": "c4", "n": c["n"], "m": c["m"], "graph_seed": bench.GRAPH_SEED,
           "indptr_sha256": hashlib.sha256(g.indptr.tobytes()).hexdigest(),
           "indices_sha256": hashlib.sha256(g.indices.tobytes()).hexdigest(),
           "max_degree": int(deg.max()), "isolated": int((deg == 0).sum()),
           "generator": "oracle ob_rmat_par", "gen_s": round(time.time() - t0, 1)}
    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "c4_csr.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(out)


if __name__ == "__main__":
    main()
