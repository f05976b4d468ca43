"""CPU: pin the plain-C restatement (oracle/coopbatch_oracle.c) against the
golden vectors produced by the reference's OWN compiled code
(tests/golden/make_golden.py). These run without a GPU and without
/root/reference (the fixtures are committed)."""
import hashlib
import os

import numpy as np
import pytest

from oracle import oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden", "reference_golden.npz")


@pytest.fixture(scope="module")
def G():
    return np.load(GOLD)


@pytest.fixture(scope="module")
def pl(G):
    return O.CSR(G["pl_indptr"], G["pl_indices"])


def test_mix64_and_hash_bits(G):
    L = O.lib()
    got = [L.ob_mix64(int(x)) for x in G["mix64_in"]]
    assert np.array_equal(np.array(got, np.uint64), G["mix64_out"])
    for s, ids, n, want in zip(G["hash_seed"], G["hash_ids"], G["hash_nids"], G["hash_out"]):
        assert O.hash_bits(int(s), ids[:n].tolist()) == int(want)


def test_phi_inverse_phi_bitwise(G):
    """FP64 Phi / Phi^-1 (rng.cpp:7-52): same libm, same evaluation order ->
    bit-identical doubles."""
    L = O.lib()
    assert np.array_equal(np.array([L.ob_phi(float(x)) for x in G["phi_in"]]), G["phi_out"])
    assert np.array_equal(np.array([L.ob_inverse_phi(float(p)) for p in G["iphi_in"]]),
                          G["iphi_out"])
    assert np.array_equal(np.array([L.ob_normal_from_bits(int(b)) for b in G["nfb_in"]]),
                          G["nfb_out"])


def test_seed_schedule(G):
    for kappa in (1, 4, O.KAPPA_INF):
        s = O.make_sched(kappa, 77)
        seq = []
        for _ in range(20):
            seq.append([s.kappa, s.z1, s.z2, s.iteration])
            s = O.advance(s)
        assert np.array_equal(np.array(seq, np.uint64), G[f"sched_k{min(kappa, 999)}"])


def test_smoothed_labor_variates(G):
    L = O.lib()
    s = O.make_sched(4, 5)
    got = []
    for _ in range(6):
        for t in (0, 1, 17, 4095):
            got.append(L.ob_labor_variate(O.Sched(s.kappa, s.z1, s.z2, s.iteration), 1, t))
        s = O.advance(s)
    assert np.array_equal(np.array(got), G["labor_variates_k4"])


def test_partition_random(G):
    assert np.array_equal(O.partition_random(1000, 4, 3), G["owner_1000_p4_s3"])


@pytest.mark.parametrize("kname,kind", [("full", O.FULL), ("ns", O.NS), ("labor", O.LABOR0)])
@pytest.mark.parametrize("kappa", [1, 4])
def test_expand(G, pl, kname, kind, kappa):
    sc = O.advance(O.advance(O.make_sched(kappa, 11)))
    st = O.expand(pl, G["pl_seeds"], 3, kind, 3, sc)
    for l, b in enumerate(st):
        for k in ("dst", "src", "edges", "dst_pos"):
            assert np.array_equal(b[k], G[f"exp_{kname}_k{kappa}_l{l}_{k}"]), (l, k)


def test_coop_sample(G, pl):
    owner = G["coop_owner"]
    per_pe = [G[f"coop_seeds_p{p}"] for p in range(4)]
    assert all(np.array_equal(a, b) for a, b in zip(per_pe, O.draw_coop_seeds(owner, 4, 12, 9, 0)))
    res = O.coop_sample(pl, owner, 4, per_pe, 3, O.LABOR0, 4, O.plain_sched(21))
    for p in range(4):
        assert np.array_equal(res["owner_sets"][p], G[f"coop_owner_set_p{p}"])
        for l in range(3):
            for k in ("src", "edges"):
                assert np.array_equal(res["stacks"][p][l][k], G[f"coop_p{p}_l{l}_{k}"])
    for l in range(3):
        e = res["exchanges"][l]
        assert np.array_equal(e["send_counts"], G[f"coop_x{l}_send_counts"])
        assert np.array_equal(np.concatenate(e["loc_row"]), G[f"coop_x{l}_loc_row"])
        assert np.array_equal(np.concatenate(e["loc_part"]), G[f"coop_x{l}_loc_part"])


def test_feature_rows(G):
    got = O.feature_rows(17, 5, "f64", G["feat_ids"])
    assert np.array_equal(got, G["feat_rows_f64"])
    # one rounding to fp32 / fp16 equals rounding the reference's f64 values
    assert np.array_equal(O.feature_rows(17, 5, "f32", G["feat_ids"]),
                          G["feat_rows_f64"].astype(np.float32))
    assert np.array_equal(O.feature_rows(17, 5, "f16", G["feat_ids"]),
                          G["feat_rows_f64"].astype(np.float16))


def test_lru(G):
    lru = O.Lru(8)
    got = np.array([lru.access(int(k)) for k in G["lru_trace"]], np.uint8)
    assert np.array_equal(got, G["lru_miss_cap8"])


@pytest.mark.parametrize("kappa", [1, 4, O.KAPPA_INF])
def test_dependent_experiment(G, pl, kappa):
    r = O.dependent_experiment_restated(pl, kappa, 32, 12, 60, O.LABOR0, 4, 2, 8, 4, 5)
    assert np.array_equal(r["fingerprint"], G[f"dep_k{min(kappa, 999)}_fingerprint"])
    assert np.array_equal(r["s_l"], G[f"dep_k{min(kappa, 999)}_s_l"])


def test_rmat_digest(G):
    rm = O.rmat(1 << 12, 1 << 15, 7)
    d = hashlib.sha256(rm.indptr.tobytes() + rm.indices.tobytes()).digest()
    assert np.array_equal(np.frombuffer(d, np.uint8), G["rmat_4096_32768_7_sha"])
    # structural: simple graph, in-range, exactly m edges, CSR order = attempt order
    assert rm.indices.max() < rm.n and rm.m == 1 << 15
    for v in range(0, rm.n, 97):
        nb = rm.indices[rm.indptr[v]:rm.indptr[v + 1]]
        assert len(set(nb.tolist())) == len(nb) and v not in nb.tolist()


@pytest.mark.parametrize("n,m,seed", [(1 << 12, 1 << 15, 7), (1 << 16, 1 << 20, 42),
                                      (5000, 3_000_000, 3), (3, 6, 1), (100, 0, 1)])
def test_rmat_parallel_equals_sequential(n, m, seed):
    """ob_rmat_par (bucketed, multi-threaded; builds the c4 graph for the
    reference arm and tests/golden/c4_csr.json) == the sequential ob_rmat."""
    a = O.rmat(n, m, seed, parallel=False)
    b = O.rmat(n, m, seed, parallel=True)
    assert np.array_equal(a.indptr, b.indptr) and np.array_equal(a.indices, b.indices)
