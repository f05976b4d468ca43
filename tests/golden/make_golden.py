"""Generate tests/golden/reference_golden.npz from the reference's OWN code.

Run in the build container (where /root/reference exists and
oracle/_ref/libcoopbatch_ref.so was compiled from its sources by
oracle/Makefile):

    python tests/golden/make_golden.py

Every array below is produced by calling the compiled reference
(coopbatch::mix64 / hash_bits / phi / inverse_phi / SeedSchedule /
partition_random / generate_powerlaw / expand / coop_sample /
FeatureStore / LruCache / run_dependent_experiment) through the
oracle/ref_capi.cpp shim. The CPU tests pin the plain-C restatement
(oracle/coopbatch_oracle.c) against these vectors; the GPU tests pin the
CUDA path against the restatement. The R-MAT generator is this repo's own
spec (the reference has none); its golden digest pins the restatement.
"""
import hashlib
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_golden.npz")


def main():
    R = "reference"
    g = {}
    # --- rng.hpp:17-48 -------------------------------------------------------
    xs = np.array([0, 1, 2, 42, 0xDEADBEEF, (1 << 63) + 5, (1 << 64) - 1], dtype=np.uint64)
    L = O.lib(R)
    g["mix64_in"] = xs
    g["mix64_out"] = np.array([L.rf_mix64(int(x)) for x in xs], dtype=np.uint64)
    tuples = [(7, [1]), (42, [2, 0, 17]), (0, [9, 123, 4]), (2**40 + 3, [12, 1]),
              (99, [8, 5, 77]), (1234, [13, 5, 0]), (5, [7, 1999])]
    g["hash_seed"] = np.array([t[0] for t in tuples], dtype=np.uint64)
    g["hash_ids"] = np.array([t[1] + [0] * (3 - len(t[1])) for t in tuples], dtype=np.uint64)
    g["hash_nids"] = np.array([len(t[1]) for t in tuples], dtype=np.int32)
    g["hash_out"] = np.array([O.hash_bits(s, ids, R) for s, ids in tuples], dtype=np.uint64)
    # --- rng.cpp:7-52 --------------------------------------------------------
    px = np.array([-8.0, -3.3, -1.0, -0.25, 0.0, 0.5, 1.7, 4.2, 7.9])
    g["phi_in"], g["phi_out"] = px, np.array([L.rf_phi(float(x)) for x in px])
    pp = np.array([1e-12, 0.001, 0.02, 0.02425, 0.1, 0.5, 0.77, 0.97575, 0.999, 1 - 1e-9])
    g["iphi_in"], g["iphi_out"] = pp, np.array([L.rf_inverse_phi(float(p)) for p in pp])
    bits = np.array([O.hash_bits(3, [i]) for i in range(16)], dtype=np.uint64)
    g["nfb_in"], g["nfb_out"] = bits, np.array([L.rf_normal_from_bits(int(b)) for b in bits])
    # --- SeedSchedule (rng.cpp:69-86) -----------------------------------------
    for kappa in (1, 4, O.KAPPA_INF):
        s = O.make_sched(kappa, 77, R)
        seq = []
        for _ in range(20):
            seq.append([s.kappa, s.z1, s.z2, s.iteration])
            s = O.advance(s, R)
        g[f"sched_k{min(kappa, 999)}"] = np.array(seq, dtype=np.uint64)
    # smoothed LABOR variates (samplers.cpp:112-129) at several contributions
    var = []
    s = O.make_sched(4, 5, R)
    for it in range(6):
        for t in (0, 1, 17, 4095):
            var.append(L.rf_labor_variate(O.Sched(s.kappa, s.z1, s.z2, s.iteration), 1, t))
        s = O.advance(s, R)
    g["labor_variates_k4"] = np.array(var)
    # --- partition_random (partition.cpp:10-20) --------------------------------
    g["owner_1000_p4_s3"] = O.partition_random(1000, 4, 3, R)
    # --- graph + sampling (samplers.cpp, coop.cpp) ----------------------------
    pg = O.generate_powerlaw(500, 6, 0.5, 3)
    g["pl_indptr"], g["pl_indices"] = pg.indptr, pg.indices
    seeds = np.array([5, 9, 100, 317, 499, 0, 250, 251], dtype=np.uint32)
    g["pl_seeds"] = seeds
    for kind, kname in ((O.FULL, "full"), (O.NS, "ns"), (O.LABOR0, "labor")):
        for kappa in (1, 4):
            sc = O.advance(O.advance(O.make_sched(kappa, 11, R), R), R)
            st = O.expand(pg, seeds, 3, kind, 3, sc, impl=R)
            for l, b in enumerate(st):
                for k in ("dst", "src", "edges", "dst_pos"):
                    g[f"exp_{kname}_k{kappa}_l{l}_{k}"] = b[k]
    owner = O.partition_random(pg.n, 4, 9, R)
    per_pe = O.draw_coop_seeds(owner, 4, 12, 9, 0)
    g["coop_owner"] = owner
    for p in range(4):
        g[f"coop_seeds_p{p}"] = per_pe[p]
    res = O.coop_sample(pg, owner, 4, per_pe, 3, O.LABOR0, 4, O.plain_sched(21), impl=R)
    for p in range(4):
        g[f"coop_owner_set_p{p}"] = res["owner_sets"][p]
        for l in range(3):
            for k in ("src", "edges"):
                g[f"coop_p{p}_l{l}_{k}"] = res["stacks"][p][l][k]
    for l in range(3):
        e = res["exchanges"][l]
        g[f"coop_x{l}_send_counts"] = e["send_counts"]
        g[f"coop_x{l}_loc_row"] = np.concatenate(e["loc_row"])
        g[f"coop_x{l}_loc_part"] = np.concatenate(e["loc_part"])
    # --- FeatureStore (coop.cpp:359-388) ---------------------------------------
    fs = O.RefFeatureStore(pg.n, 5, 17)
    ids = np.array([0, 3, 499, 250], dtype=np.uint32)
    g["feat_ids"], g["feat_rows_f64"] = ids, fs.load_rows(ids)
    # --- LruCache (cache.cpp:8-32) ----------------------------------------------
    trace = np.array([O.hash_bits(1, [i]) % 37 for i in range(400)], dtype=np.uint32)
    lru = O.Lru(8, R)
    g["lru_trace"] = trace
    g["lru_miss_cap8"] = np.array([lru.access(int(k)) for k in trace], dtype=np.uint8)
    # --- run_dependent_experiment (cache.cpp:137-208) -------------------------
    for kappa in (1, 4, O.KAPPA_INF):
        r = O.dependent_experiment(pg, 2, kappa, 32, 12, 60, O.LABOR0, 4, 2, 8, 4, 5)
        g[f"dep_k{min(kappa, 999)}_fingerprint"] = r["fingerprint"]
        g[f"dep_k{min(kappa, 999)}_s_l"] = r["s_l"]
    # --- R-MAT (this repo's spec; the reference has no R-MAT) ------------------
    rm = O.rmat(1 << 12, 1 << 15, 7)
    g["rmat_4096_32768_7_sha"] = np.frombuffer(
        hashlib.sha256(rm.indptr.tobytes() + rm.indices.tobytes()).digest(), dtype=np.uint8)
    np.savez_compressed(OUT, **g)
    print(f"wrote {OUT}: {len(g)} arrays")


if __name__ == "__main__":
    main()
