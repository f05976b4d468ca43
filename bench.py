#!/usr/bin/env python
"""Benchmark of the cooperative-minibatching hot path on B200.

Metric (BASELINE.json): seed vertices/sec of one minibatch step =
3-layer LABOR-0 sample + dedup/relabel (+ owner exchange) + input-feature
gather, plus feature GB/s. Headline workload: config 4, the
ogbn-papers100M-shaped R-MAT (111M V / 1.6B E, 128 fp16 rows) that north_star
targets and that fits one B200 (`--config` picks another BASELINE config).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4]
  python bench.py --impl reference ...   # the reference's own CPU path

One process per GPU (torchrun for N>1).
  N = 1 : independent minibatches of 1024 seeds, S = 8 in flight (one CUDA
          graph + stream each); `latency_ms_per_step` is one batch at a time
          with L2 flushed (512 MiB write + 256 MiB read) before every step;
          `latency_unflushed_ms_per_step` the same without the flush.
          `value` is not flushed between steps: the inputs (6.5 GB CSR +
          28 GB table at c4) are far larger than the 126 MB L2.
  N > 1 : the cooperative step (one part per GPU, per-layer owner exchange
          over peer memory, owners stage their requested rows and requesters
          pull them; the whole step one CUDA graph per rank with device
          barriers; weak scaling, 1024 seeds per GPU). See DESIGN.md
          §Multi-GPU.

value  : device time (CUDA events, max over ranks), inputs resident in HBM.
e2e    : through the C-ABI with host buffers: H2D of the seeds + variate keys
         from pinned memory, sample + gather, and the whole batch result
         (every layer's blocks and the gathered rows) written to pinned host
         memory, every step; wall clock.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import subprocess
import sys
import threading
import math
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "seed vertices/sec (sample+dedup+gather, 3-layer) at 1/2/4/8 B200; feature GB/s"

CONFIGS = {
    "c1": dict(workload="c1: R-MAT 2^16 V / 2^20 E, NS fanout 10, 3 layers, batch 1024, "
                        "feat 128 fp32", n=1 << 16, m=1 << 20, kind="ns", fanouts=[10, 10, 10],
               batch=1024, dim=128, dtype="f32"),
    "c2": dict(workload="c2: ogbn-products-shaped R-MAT (2,449,029 V / 61,859,140 E), "
                        "LABOR-0 fanout 10, 3 layers, batch 1024/GPU, feat 100 fp32",
               n=2449029, m=61859140, kind="labor0", fanouts=[10, 10, 10], batch=1024, dim=100,
               dtype="f32"),
    "c3": dict(workload="c3: reddit-shaped dense R-MAT (232,965 V / 114,615,892 E), LABOR-0 "
                        "fanout 10, 3 layers, batch 1024, feat 602 fp32",
               n=232965, m=114615892, kind="labor0", fanouts=[10, 10, 10], batch=1024, dim=602,
               dtype="f32"),
    "c4": dict(workload="c4: ogbn-papers100M-shaped R-MAT (111,059,956 V / 1,615,685,872 E), "
                        "LABOR-0 fanout 10, 3 layers, batch 1024/GPU, feat 128 fp16",
               n=111059956, m=1615685872, kind="labor0", fanouts=[10, 10, 10], batch=1024,
               dim=128, dtype="f16"),
    "c5": dict(workload="c5: mag240M-shaped R-MAT (244,160,499 V / 1,728,364,232 E), "
                        "2-layer fanout 25/15, batch 1024/GPU, feat 768 fp16",
               n=244160499, m=1728364232, kind="labor0", fanouts=[25, 15], batch=1024, dim=768,
               dtype="f16"),
}
GRAPH_SEED = 42
CSV_ROWS: dict = {}  # per-step report rows for --csv-dir (reports.py)
FEAT_SEED = 7
RUN_SEED = 1234


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def ncu_traffic(cfg_name: str, seeds_step: int) -> dict:
    """DRAM traffic per launch of the roofline kernels, measured in this run:
    a child process (`bench.py --probe`) samples the same batch the
    per-kernel profile uses (step `seeds_step`) eagerly and gathers its rows,
    under `ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum` (cold
    cache, serialised launches). Returns {kernel: bytes} for the last layer's
    labor_mark and the gather, or {"error": ...}."""
    import csv
    import shutil
    import tempfile
    ncu = shutil.which("ncu") or "/usr/local/cuda/bin/ncu"
    if not os.path.exists(ncu):
        return {"error": "ncu not found"}
    with tempfile.TemporaryDirectory() as td:
        log = os.path.join(td, "traffic.csv")
        cmd = [ncu, "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum,"
               "gpu__time_duration.sum", "--clock-control", "none", "-k",
               "regex:labor_mark_kernel|gather_kernel", "--csv", "--log-file", log,
               sys.executable, os.path.abspath(__file__), "--probe", "--config", cfg_name,
               "--probe-step", str(seeds_step)]
        try:
            r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
        except Exception as e:  # noqa: BLE001 - report, never fake
            return {"error": f"ncu run failed: {e}"[:200]}
        if r.returncode != 0 or not os.path.exists(log):
            return {"error": f"ncu rc={r.returncode}: {(r.stderr or r.stdout)[-200:]}"}
        launches: dict = {}
        with open(log) as f:
            rows = [x for x in csv.reader(f)]
        hi = next(i for i, x in enumerate(rows) if "Metric Name" in x)
        h = rows[hi]
        iid, ik, im, iv = (h.index("ID"), h.index("Kernel Name"), h.index("Metric Name"),
                           h.index("Metric Value"))
        for x in rows[hi + 1:]:
            if len(x) <= iv:
                continue
            e = launches.setdefault(int(x[iid]), {"kernel": x[ik]})
            e[x[im]] = float(x[iv].replace(",", ""))
    order = [launches[k] for k in sorted(launches)]
    marks = [e for e in order if "labor_mark" in e["kernel"]]
    gathers = [e for e in order if "gather_kernel" in e["kernel"]]
    out = {"how": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum "
                  "--clock-control none (bench.py --probe child, same batch)"}
    if marks:
        e = marks[-1]
        out["labor_mark_last_layer"] = e["dram__bytes_read.sum"] + e["dram__bytes_write.sum"]
        out["labor_mark_ncu_us"] = e["gpu__time_duration.sum"] / 1e3
    if gathers:
        e = gathers[-1]
        out["gather"] = e["dram__bytes_read.sum"] + e["dram__bytes_write.sum"]
        out["gather_ncu_us"] = e["gpu__time_duration.sum"] / 1e3
    return out


def run_probe(args, cfg):
    """--probe: one eager batch (step args.probe_step's seeds and schedule,
    the batch the per-kernel profile times) + its gather, for ncu_traffic."""
    import paper_2310_12403_b200 as cb
    from paper_2310_12403_b200.seeds import draw_from_pool
    kind = {"labor0": cb.SamplerKind.kLabor0, "ns": cb.SamplerKind.kNs,
            "full": cb.SamplerKind.kFull}[cfg["kind"]]
    L, b = len(cfg["fanouts"]), cfg["batch"]
    g = cb.Graph.generate_rmat(cfg["n"], cfg["m"], GRAPH_SEED, device=0)
    store = cb.FeatureStore.synth(g, cfg["dim"], FEAT_SEED, cfg["dtype"])
    scfg = cb.SamplerConfig(kind, fanouts=cfg["fanouts"])
    i = args.probe_step
    seeds = draw_from_pool(np.arange(cfg["n"], dtype=np.uint32), b, RUN_SEED,
                           cb.hash_bits(i, [0]))
    sched = cb.SeedSchedule.make(1, RUN_SEED)
    for _ in range(i):
        sched = cb.schedule_advance(sched)
    plan = cb.Plan(g, None, L, scfg, b)
    plan.sample([seeds], sched, cb.MODE_INDEP, sync=True)
    plan.gather(store)
    plan.synchronize()
    print(json.dumps({"probe": [plan.layer_sizes(0, l) for l in range(L)]}))


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class ClockSampler:
    """NVML sampling of SM clocks + throttle reasons during the timed region."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, device: int):
        self.samples, self.reasons, self.ok = [], set(), False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max = None
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        med = float(np.median(self.samples)) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


# ------------------------------------------------------------ CPU baseline --
def cpu_reference_leg(cfg, csr, budget_s: float, parts_per_step: int | None = None,
                      max_steps: int | None = None, coop_parts: int = 0):
    """Time the reference's own stock path on this host's cores (oracle/_ref,
    the reference compiled from its sources): indep_sample over P parts of
    `batch` seeds (the reference parallelises over parts, coop.cpp:115-117) +
    per-part FeatureStore::load_rows; or, with coop_parts = P > 1,
    coop_sample over P parts + load_rows of the owner sets +
    all_to_all_forward (coop.cpp:445-467). When the f64 FeatureStore would not
    fit (c4: 113 GB), rows are computed from FeatureStore::synth's formula
    instead of copied. Returns (seeds/s, cores, sample
    description, per-step seconds list)."""
    from oracle import oracle as O
    threads = os.cpu_count() or 1
    coop = coop_parts > 1
    P = coop_parts if coop else (parts_per_step or threads)
    rg = O.RefGraph(csr)
    onfly = csr.n * cfg["dim"] * 8 > (8 << 30)
    t0 = time.time()
    fs = None if onfly else O.RefFeatureStore(csr.n, cfg["dim"], FEAT_SEED)
    synth_s = time.time() - t0
    kind = {"labor0": O.LABOR0, "ns": O.NS, "full": O.FULL}[cfg["kind"]]
    sched = O.make_sched(1, RUN_SEED)
    L = len(cfg["fanouts"])
    if len(set(cfg["fanouts"])) != 1:
        raise SystemExit("reference leg: per-layer fanouts need the sample_block loop")
    if coop:
        owner = O.partition_random(csr.n, P, RUN_SEED)
        members = O.part_members(owner, P)
    else:
        pool = np.arange(csr.n, dtype=np.uint32)
    steps, seeds_done, spent, per_step = 0, 0, 0.0, []
    while (steps == 0 or spent < budget_s) and (max_steps is None or steps < max_steps):
        if coop:
            per_pe = [O.draw_from_pool(members[p], cfg["batch"], RUN_SEED,
                                       O.hash_bits(steps, [p])) for p in range(P)]
        else:
            per_pe = [O.draw_from_pool(pool, cfg["batch"], RUN_SEED, O.hash_bits(steps, [p]))
                      for p in range(P)]
        mode = 0 if coop else 1
        own = owner if coop else None
        if onfly:
            ts, tg, rows = O.reference_step_onfly(rg, FEAT_SEED, cfg["dim"], mode, own, P,
                                                  per_pe, L, kind, cfg["fanouts"][0], sched)
        else:
            ts, tg, rows = O.reference_step(rg, fs, mode, own, P, per_pe, L, kind,
                                            cfg["fanouts"][0], sched)
        per_step.append(ts + tg)
        spent += ts + tg
        seeds_done += sum(len(x) for x in per_pe)
        sched = O.advance(sched)
        steps += 1
    what = (f"coop_sample over {P} parts x {cfg['batch']} seeds + load_rows(owner_sets) + "
            "all_to_all_forward" if coop else
            f"indep_sample over {P} parts x {cfg['batch']} seeds + per-part load_rows")
    rows_how = ("rows computed from FeatureStore::synth's formula with the reference's "
                "hash (the f64 store would be "
                f"{csr.n * cfg['dim'] * 8 / 1e9:.0f} GB), parallel over parts"
                if onfly else f"f64 FeatureStore rows (synth {synth_s:.1f}s excluded)")
    desc = (f"{steps} step(s) x {what} (reference parallel_for over parts, "
            f"COOPBATCH_THREADS={threads}); {rows_how}")
    return seeds_done / spent, min(P, threads), desc, per_step


def run_reference(args, cfg):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from oracle import oracle as O
    t0 = time.time()
    csr = O.rmat(cfg["n"], cfg["m"], GRAPH_SEED)
    gen_s = time.time() - t0
    threads = os.cpu_count() or 1
    coop_parts = world if world > 1 else 0
    # probe one batch to size the per-step sample
    _, _, _, probe = cpu_reference_leg(cfg, csr, 0.0, parts_per_step=1, max_steps=1,
                                       coop_parts=coop_parts)
    per_batch = max(probe[0], 1e-3)
    budget = 120.0
    # parts run in parallel over the host threads (coop.cpp:115-117): one
    # wave of `threads` parts costs about one probe batch, so every step uses
    # all the threads, with up to 4 waves while the run stays within budget
    waves = int(max(1, min(4, budget / max(1, args.steps + args.warmup) / per_batch)))
    P = threads * waves
    value, cores, desc, per_step = cpu_reference_leg(
        cfg, csr, float("inf"), parts_per_step=P, max_steps=args.warmup + args.steps,
        coop_parts=coop_parts)
    timed = per_step[args.warmup:] or per_step
    seeds = (coop_parts or P) * cfg["batch"] * len(timed)
    v = seeds / sum(timed)
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "seeds/s",
        "n_gpus": world, "steps": len(timed), "warmup": args.warmup,
        "ms_per_step": 1000 * sum(timed) / len(timed), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64 rows / u32 ids",
        "data": "synthetic (hash-keyed R-MAT, hashed features)",
        "config": {"workload": cfg["workload"],
                   "mode": (f"cooperative (P={world} parts)" if coop_parts else
                            f"indep ({P} independent minibatches per step)"),
                   "graph_gen_s": round(gen_s, 1),
                   "graph_gen": "oracle R-MAT on the host cores (ob_rmat_par)"},
        "cpu_baseline": {"value": v, "unit": "seeds/s", "cores": cores, "kind": "reference",
                         "sample": desc},
        "e2e": {"value": v, "unit": "seeds/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------ concavity evidence --
def concavity_evidence(cb, g, scfg, L, b, row_bytes, dev, parts=(1, 2, 4, 8)):
    """The paper's work comparison at equal global batch (acceptance.cpp:
    270-300): P parts of b seeds (cli.cpp:210-214 draws), cooperative
    (coop_sample: per-owner input sets |S^L_p| after the exchange) vs
    independent (the same global batch split round-robin, indep_sample).
    All P parts run on this one GPU (the reference's simulated PEs)."""
    import torch

    from paper_2310_12403_b200.seeds import coop_seeds
    out = []
    sched = cb.SeedSchedule.make(1, RUN_SEED)
    for P in parts:
        pm = cb.partition_random(g, P, RUN_SEED)
        seeds = coop_seeds(pm.members(), b, RUN_SEED, 0)
        plan = cb.Plan(g, pm, L, scfg, b)
        plan.sample(seeds, sched, cb.MODE_COOP)
        # device time of one cooperative step of P parts on this GPU: the
        # captured batch (sampling + per-layer rendezvous), replayed
        plan.capture(np.arange(P + 1, dtype=np.uint64) * b, sched, cb.MODE_COOP, None)
        st = torch.cuda.ExternalStream(plan.stream, device=torch.device(f"cuda:{dev}"))
        d = torch.from_numpy(np.concatenate(seeds).view(np.int32)).to(f"cuda:{dev}")
        tms = []
        for _ in range(4):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            plan.replay(d.data_ptr(), sched, True, 1)
            e1.record(st)
            plan.synchronize()
            tms.append(e0.elapsed_time(e1))
        coop_ms = float(np.mean(tms[1:]))
        CSV_ROWS.setdefault("run", []).append(
            (f"coop_P{P}", cb.step_metrics(plan, cb.MODE_COOP, row_bytes)))
        c_s3 = sum(len(plan.owner_set(p)) for p in range(P))
        c_work = sum(plan.layer_sizes(p, l)["n_edges"] for p in range(P) for l in range(L))
        c_comm = sum(plan.exchange(l).total_communicated() for l in range(L))
        union = np.concatenate(seeds)
        chunks = [union[i::P] for i in range(P)]
        ip = cb.Plan(g, None, L, scfg, max(len(c) for c in chunks))
        i_s3 = i_work = 0
        for c in chunks:
            ip.sample([c], sched, cb.MODE_INDEP)
            i_s3 += ip.layer_sizes(0, L - 1)["n_src"]
            i_work += sum(ip.layer_sizes(0, l)["n_edges"] for l in range(L))
        gb = P * b
        out.append({"P": P, "global_batch": gb,
                    "coop": {"input_vertices_per_seed": c_s3 / gb, "edges_per_seed": c_work / gb,
                             "feature_bytes_per_seed": c_s3 * row_bytes / gb,
                             "ids_exchanged_per_seed": c_comm / gb,
                             "step_ms_one_gpu_graph": round(coop_ms, 4)},
                    "indep": {"input_vertices_per_seed": i_s3 / gb, "edges_per_seed": i_work / gb,
                              "feature_bytes_per_seed": i_s3 * row_bytes / gb}})
        del plan, ip, pm
    return out


# ---------------------------------------------------------- scale evidence --
def scale_evidence(cb, dev, name="c2", steps=20, parts=(1, 8)):
    """Another BASELINE config on one B200 (c2 products-shaped when the
    headline is c4): one batch at a time (CUDA graphs, L2 flushed, events),
    the gather's roofline, and cooperative vs independent per-seed work at
    P = 1 and 8 (simulated parts on this GPU)."""
    import torch

    c = CONFIGS[name]
    t0 = time.time()
    g = cb.Graph.generate_rmat(c["n"], c["m"], GRAPH_SEED, device=dev)
    gen_s = time.time() - t0
    store = cb.FeatureStore.synth(g, c["dim"], FEAT_SEED, c["dtype"])
    scfg = cb.SamplerConfig(cb.SamplerKind.kLabor0, fanouts=c["fanouts"])
    L, b = len(c["fanouts"]), c["batch"]
    plan = cb.Plan(g, None, L, scfg, b)
    pool = np.arange(c["n"], dtype=np.uint32)
    from paper_2310_12403_b200.seeds import draw_from_pool
    seeds = [draw_from_pool(pool, b, RUN_SEED, cb.hash_bits(s, [0])) for s in range(steps + 3)]
    scheds = [cb.SeedSchedule.make(1, RUN_SEED)]
    for _ in range(steps + 3):
        scheds.append(cb.schedule_advance(scheds[-1]))
    plan.sample([seeds[0]], scheds[0], cb.MODE_INDEP, sync=True)
    plan.capture(np.array([0, b], np.uint64), scheds[0], cb.MODE_INDEP, store)
    st = torch.cuda.ExternalStream(plan.stream, device=torch.device(f"cuda:{dev}"))
    d = torch.from_numpy(np.stack(seeds).view(np.int32)).to(f"cuda:{dev}")
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=f"cuda:{dev}")
    clean = torch.empty(64 << 20, dtype=torch.int32, device=f"cuda:{dev}")

    def flush_l2():  # same as the headline: 512 MiB write, then 256 MiB read
        with torch.cuda.stream(st):
            flush.zero_()
            clean.sum()
    ms, gms = [], []
    for i in range(steps + 3):
        flush_l2()
        e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        e[0].record(st)
        plan.replay(d.data_ptr() + i * b * 4, scheds[i], True, 3)
        e[1].record(st)
        flush_l2()
        e[2].record(st)
        plan.gather(store)
        e[3].record(st)
        plan.synchronize()
        if i >= 3:
            ms.append(e[0].elapsed_time(e[1]))
            gms.append(e[2].elapsed_time(e[3]))
    rows = plan.layer_sizes(0, L - 1)["n_src"]
    store_row_bytes = store.row_bytes
    gbytes = rows * (2 * store.row_bytes + 4)
    peak, _ = peaks()
    out = {"workload": c["workload"], "graph_gen_s": round(gen_s, 2),
           "seeds_per_s": b / (np.mean(ms) / 1e3), "ms_per_step": float(np.mean(ms)),
           "gather": {"ms": float(np.mean(gms)), "rows": rows,
                      "achieved_gbs": gbytes / (np.mean(gms) / 1e3) / 1e9,
                      "frac": gbytes / (np.mean(gms) / 1e3) / 1e9 / peak},
           "per_layer": [plan.layer_sizes(0, l) for l in range(L)]}
    del plan, store
    out["concavity"] = concavity_evidence(cb, g, scfg, L, b, store_row_bytes, dev, parts=parts)
    del g
    return out


# ------------------------------------------------------ c5 batch sweep ------
def batch_sweep_evidence(cb, dev, batches=(1024, 4096, 16384, 65536), steps=10):
    """Config 5's batch sweep on one B200: mag240M-shaped R-MAT (244M V /
    1.73B E), 2-layer LABOR-0 fanout 25/15. The 768-dim fp16 table (375 GB)
    does not fit one GPU, so this sweep times sampling + dedup only and
    reports the feature bytes the batch would fetch (rows x 1536 B)."""
    import torch

    c = CONFIGS["c5"]
    t0 = time.time()
    g = cb.Graph.generate_rmat(c["n"], c["m"], GRAPH_SEED, device=dev)
    gen_s = time.time() - t0
    scfg = cb.SamplerConfig(cb.SamplerKind.kLabor0, fanouts=c["fanouts"])
    L = len(c["fanouts"])
    rng = np.random.default_rng(RUN_SEED)
    out = {"workload": c["workload"] + " (sampling + dedup only)", "graph_gen_s": round(gen_s, 2),
           "sweep": []}
    for b in batches:
        plan = cb.Plan(g, None, L, scfg, b)
        seeds = [np.sort(rng.choice(c["n"], b, replace=False)).astype(np.uint32)
                 for _ in range(steps + 2)]
        sched = cb.SeedSchedule.make(1, RUN_SEED)
        plan.sample([seeds[0]], sched, cb.MODE_INDEP, sync=True)
        plan.capture(np.array([0, b], np.uint64), sched, cb.MODE_INDEP, None)
        st = torch.cuda.ExternalStream(plan.stream, device=torch.device(f"cuda:{dev}"))
        d = torch.from_numpy(np.stack(seeds).view(np.int32)).to(f"cuda:{dev}")
        ms, rows = [], []
        for i in range(steps + 2):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            plan.replay(d.data_ptr() + i * b * 4, sched, True, 1)
            e1.record(st)
            plan.synchronize()
            sched = cb.schedule_advance(sched)
            if i >= 2:
                ms.append(e0.elapsed_time(e1))
                rows.append(plan.layer_sizes(0, L - 1)["n_src"])
        CSV_ROWS.setdefault("curve", []).append(
            (b, float(np.mean(rows)), float(np.std(rows) / np.sqrt(len(rows))),
             float(np.mean(rows)) / b))
        out["sweep"].append({"batch": b, "ms_per_batch": float(np.mean(ms)),
                             "seeds_per_s": b / (float(np.mean(ms)) / 1e3),
                             "input_vertices_per_seed": float(np.mean(rows)) / b,
                             "feature_bytes_per_seed": float(np.mean(rows)) * 1536 / b})
        del plan, d
    del g
    return out


def mark_roofline(prof_ms, prof_sizes, L, scfg, peak, peak_kind, traffic):
    """The dominant kernel: labor_mark of the last layer (c4: ~40% of a
    batch), timed by the in-graph event profile of one batch (mean of the
    replays, L2 flushed before each). Algorithmic bytes per launch (SURVEY
    §8(d)): 4 B per scanned position (the neighbour id) + 4 B per 32 positions
    (keep word) + 8 B per kept edge (staged pair). `traffic` is the same
    launch's DRAM bytes measured by ncu in this run (ncu_traffic)."""
    import math as _m
    if int(scfg.kind) != 2 or len(prof_ms) != 3 * L + 3:
        return None
    i = 3 * (L - 1) + 2
    s = prof_sizes[L - 1]
    nbytes = 4 * s["scan_total"] + 4 * _m.ceil(s["scan_total"] / 32) + 8 * s["n_edges"]
    t = prof_ms[i] / 1e3
    return {"bound": "hbm", "kernel": "labor_mark_kernel (last layer)",
            "achieved": nbytes / t / 1e9, "peak": peak, "peak_kind": peak_kind,
            "unit": "GB/s", "frac": nbytes / t / 1e9 / peak,
            "traffic": traffic.get("labor_mark_last_layer"),
            "bytes_per_launch": nbytes,
            "per_unit": "4 B per scanned position + 4 B per keep word + 8 B per kept edge",
            "ms": prof_ms[i], "positions": s["scan_total"], "kept": s["n_edges"],
            "positions_per_s": s["scan_total"] / t,
            "share_of_batch": prof_ms[i] / sum(prof_ms)}


# ------------------------------------------------------ work curves (f4) ---
def work_curve_evidence(cb, dev, cpu: bool, trials=50, layers=3, seed=49):
    """Acceptance criteria 2-3 (acceptance.cpp:137-192): E|S^3| against batch
    size 64..8192 for NS / LABOR-0 / RW (defaults k=10, o=3, p=0.5, a=100),
    50 trials per size, on the c1 R-MAT (2^16 V / 2^20 E, avg degree 16; the
    acceptance graph is a 100K-vertex degree-16 power-law graph). The trials
    of a size run as the parts of one plan (cb_sample_multi). Checks: work per
    seed nonincreasing within +1 pooled s.e., concavity_check passes. With
    `cpu`, the compiled reference's work_curve runs on the same CSR (all host
    threads) for LABOR-0 as the CPU baseline and the curves are compared."""
    import os
    c = CONFIGS["c1"]
    g = cb.Graph.generate_rmat(c["n"], c["m"], GRAPH_SEED, device=dev)
    sizes = [64 << i for i in range(8)]
    out = {"graph": "c1 R-MAT 2^16 V / 2^20 E", "sizes": sizes, "trials": trials,
           "layers": layers, "samplers": {}}
    for name, kind in (("ns", cb.SamplerKind.kNs), ("labor0", cb.SamplerKind.kLabor0),
                       ("rw", cb.SamplerKind.kRw)):
        cfg = cb.SamplerConfig(kind)
        cb.work_curve(g, cfg, sizes[:1], 2, layers, seed)  # warm-up
        t0 = time.time()
        curve = cb.work_curve(g, cfg, sizes, trials, layers, seed)
        dt = time.time() - t0
        mono = all(b.work_per_seed <= a.work_per_seed + math.sqrt(a.se_work ** 2 + b.se_work ** 2)
                   for a, b in zip(curve.points, curve.points[1:]))
        out["samplers"][name] = {
            "seconds": round(dt, 3),
            "work_per_seed": [round(p.work_per_seed, 4) for p in curve.points],
            "nonincreasing": mono, "concave": cb.concavity_check(curve).passed}
        for p in curve.points:
            CSV_ROWS.setdefault("work_curve", []).append(
                (name, p.batch_size, p.mean_sl, p.se_sl, p.work_per_seed, p.se_work))
        if cpu and name == "labor0":
            try:
                from oracle import oracle as O
                indptr, indices = g.download()
                os.environ.setdefault("COOPBATCH_THREADS", str(os.cpu_count() or 1))
                t0 = time.time()
                ref = O.work_curve_reference(O.CSR(indptr, indices), O.LABOR0, cfg.fanout, sizes,
                                             trials, layers, seed)
                rt = time.time() - t0
                got = np.array([[p.mean_sl, p.se_sl, p.work_per_seed, p.se_work]
                                for p in curve.points])
                out["samplers"][name]["cpu_baseline"] = {
                    "kind": "reference", "seconds": round(rt, 3), "cores": os.cpu_count(),
                    "equal_to_gpu": bool(np.array_equal(ref, got))}
            except Exception as e:  # noqa: BLE001 - evidence only
                out["samplers"][name]["cpu_baseline"] = {"unavailable": str(e)[:200]}
    del g
    return out


# ----------------------------------------------------- drop-in e2e evidence --
def dropin_evidence():
    """End to end through the C++ drop-in (tools/dropin_bench.cpp, built by
    tests/cpp/Makefile against libcoopbatch_core_b200): the reference's own
    coopbatch::expand + FeatureStore::load_rows (f64 rows read in place from
    the host table) with host objects in and out, on config c2."""
    exe = os.path.join(ROOT, "tests", "cpp", "_build", "dropin_bench")
    if not os.path.exists(exe):
        return {"unavailable": "tests/cpp/_build/dropin_bench not built"}
    c = CONFIGS["c2"]
    try:
        r = subprocess.run([exe, str(c["n"]), str(c["m"]), str(c["dim"]), "40"],
                           capture_output=True, text=True, timeout=600)
        d = json.loads(r.stdout.strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001 - evidence only
        return {"error": str(e)[:200]}
    d["workload"] = c["workload"] + " (rows as the reference's f64 FeatureStore)"
    d["api"] = "coopbatch::expand + FeatureStore::load_rows (reference headers, host objects)"
    return d


# ---------------------------------------------------------- kappa evidence --
def kappa_evidence(cb, dev, steps_epochs=2, kappas=(1, 4, 16, 64, 256, None)):
    """Config 3's kappa sweep (acceptance.cpp:362-390 at full scale): the
    reddit-shaped R-MAT, LABOR-0 fanout 10, 3 layers, batch 1024, smoothed
    kappa-dependent minibatches, input rows (602 fp32) fetched through the
    per-GPU LRU cache (capacity |V|/10, acceptance.cpp:368) with the feature
    table in pinned host memory: hits are served from HBM, misses cross the
    host link. Steady miss rate after one warmup epoch (cache.cpp:168-203)."""
    c = CONFIGS["c3"]
    t0 = time.time()
    g = cb.Graph.generate_rmat(c["n"], c["m"], GRAPH_SEED, device=dev)
    gen_s = time.time() - t0
    store = cb.FeatureStore.synth(g, c["dim"], FEAT_SEED, c["dtype"])
    store.set_tier(True)
    cfg = cb.SamplerConfig(cb.SamplerKind.kLabor0, fanouts=c["fanouts"])
    cap = c["n"] // 10
    spe = c["n"] // c["batch"]
    steps = steps_epochs * spe
    ref_g, ref_steps = None, 8
    try:  # the reference beside the GPU sweep (checker only, CPU)
        from oracle import oracle as O
        if O.available("reference"):
            indptr, indices = g.download()
            ref_g = O.RefGraph(O.CSR(indptr, indices))
            del indptr, indices
    except Exception:  # noqa: BLE001 - evidence only
        ref_g = None
    out = {"workload": c["workload"], "graph_gen_s": round(gen_s, 2), "cache_rows": cap,
           "feature_tier": "pinned host memory (mapped); cache rows in HBM",
           "steps": steps, "steps_per_epoch": spe, "sweep": []}
    for kappa in kappas:
        k = cb.KAPPA_INFINITY if kappa is None else kappa
        tt = time.perf_counter()
        res_stats = {"resolved": 0, "reruns": 0, "unresolved": 0}

        def on_step(step, plan):
            a, b_ = plan.resolve_stats()  # in-band decisions settled on the host
            res_stats["resolved"] += a
            res_stats["reruns"] += b_
            res_stats["unresolved"] += sum(plan.layer_sizes(0, l)["uncertified"]
                                           for l in range(len(c["fanouts"])))
        r = cb.run_dependent_experiment(g, cb.MinibatchSchedule(cb.BatchMode.kSmoothed, k,
                                                                c["batch"]), steps, cap, cfg,
                                        len(c["fanouts"]), c["dim"], 4, RUN_SEED,
                                        fingerprints=False, store=store, on_step=on_step)
        wall = time.perf_counter() - tt
        steady = r.rows[r.warmup_steps:]
        CSV_ROWS.setdefault("cache", []).append(
            (kappa, [(x.step, x.miss_rate, x.s_l, x.bytes) for x in r.rows]))
        # the same experiment through the fast CLOCK cache (same capacity)
        tt = time.perf_counter()
        rc = cb.run_dependent_experiment(g, cb.MinibatchSchedule(cb.BatchMode.kSmoothed, k,
                                                                 c["batch"]), steps, cap, cfg,
                                         len(c["fanouts"]), c["dim"], 4, RUN_SEED,
                                         fingerprints=False, store=store, cache_kind="clock")
        wall_c = time.perf_counter() - tt
        row = {
            "kappa": "inf" if kappa is None else kappa,
            "steady_miss_rate": r.steady_miss_rate,
            "clock_cache": {"steady_miss_rate": rc.steady_miss_rate,
                            "wall_ms_per_step": 1e3 * wall_c / steps},
            "input_vertices_per_seed": float(np.mean([x.s_l for x in steady])) / c["batch"],
            "storage_bytes_per_step": float(np.mean([x.bytes for x in steady])),
            "wall_ms_per_step": 1e3 * wall / steps,
            "smoothed_decisions": res_stats}
        assert res_stats["unresolved"] == 0, "unresolved smoothed decisions"
        if ref_g is not None:
            # the reference's own run_dependent_experiment (cache.cpp:137-208),
            # compiled from its sources, over the first ref_steps steps of the
            # same experiment: same |S^L| and miss bytes step by step
            tt = time.perf_counter()
            ref = O.dependent_experiment(ref_g, 2, k, c["batch"], ref_steps, cap, O.LABOR0, 10,
                                         len(c["fanouts"]), c["dim"], 4, RUN_SEED)
            ours_sl = [x.s_l for x in r.rows[:ref_steps]]
            ours_by = [x.bytes for x in r.rows[:ref_steps]]
            row["reference"] = {
                "steps": ref_steps, "cpu_s_per_step": (time.perf_counter() - tt) / ref_steps,
                "misses": [int(b) // (c["dim"] * 4) for b in ref["bytes"]],
                "equal_s_l_and_misses": bool(list(map(int, ref["s_l"])) == ours_sl and
                                             list(map(int, ref["bytes"])) == ours_by)}
        out["sweep"].append(row)
    store.set_tier(False)
    del store, g, ref_g
    return out


# ------------------------------------------------- our arm, N>1 cooperative --
def run_ours_coop(args, cfg):
    """One process per GPU, one part per rank: the cooperative step of
    coop.cpp:68-106 with the per-layer owner exchange (build_exchange,
    coop.cpp:25-64) and the feature fetch (all_to_all_forward, coop.cpp:
    145-159) as torch.distributed all-to-allv over NCCL; per-part compute is
    libcoopbatch_b200 (dist.CudaEngine). Each rank draws b seeds from the
    vertices it owns (cli.cpp:210-214). Weak scaling: b seeds per GPU."""
    import torch
    import torch.distributed as dist

    import paper_2310_12403_b200 as cb
    from paper_2310_12403_b200 import _lib
    from paper_2310_12403_b200.dist import CudaEngine, DistCoop, synth_shard
    from paper_2310_12403_b200.seeds import draw_from_pool

    rank, world, local = dist_env()
    backend = args.dist_backend
    dev = local if backend == "nccl" else 0
    torch.cuda.set_device(dev)
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{dev}"))
    else:
        dist.init_process_group("gloo")
    kind = {"labor0": cb.SamplerKind.kLabor0, "ns": cb.SamplerKind.kNs,
            "full": cb.SamplerKind.kFull}[cfg["kind"]]
    L, b = len(cfg["fanouts"]), cfg["batch"]
    t0 = time.time()
    g = cb.Graph.generate_rmat(cfg["n"], cfg["m"], GRAPH_SEED, device=dev)
    gen_s = time.time() - t0
    pm = cb.partition_random(g, world, RUN_SEED)
    mine = pm.members()[rank]
    store = synth_shard(g, pm, rank, cfg["dim"], FEAT_SEED, cfg["dtype"])
    scfg = cb.SamplerConfig(kind, fanouts=cfg["fanouts"])
    W, K = args.warmup, args.steps
    seeds_host = [draw_from_pool(mine, b, RUN_SEED, cb.hash_bits(s, [rank])) for s in range(W + K)]
    seeds_dev = [torch.from_numpy(s.view(np.int32)).to(f"cuda:{dev}") for s in seeds_host]
    scheds = [cb.SeedSchedule.make(1, RUN_SEED)]
    for _ in range(W + K):
        scheds.append(cb.schedule_advance(scheds[-1]))
    if args.exchange == "px":
        from paper_2310_12403_b200.dist import PeerCoop
        # S cooperative steps in flight (--inflight, as at N=1): S independent
        # PeerCoops, each with its own plan, exchange regions, barrier flags,
        # stream and captured graphs; step i runs on pcs[i % S]
        S = max(1, args.inflight)
        pcs = []

        def add_peer():
            pc_ = PeerCoop(g, pm, rank, L, scfg, max_seeds=b, store=store, barrier="device")
            # one eager step on every rank (kernel attributes), then the whole
            # step (L layers, device barriers, row pull) as CUDA graphs
            pc_.sample(seeds_dev[0], scheds[0])
            pc_.load_inputs()
            pc_.finish()
            pc_.capture(b, scheds[0])
            pcs.append(pc_)
        free0 = torch.cuda.mem_get_info(dev)[0]
        add_peer()
        # as many in flight as a third of the remaining HBM holds (the ranks
        # agree on the minimum), at most --inflight
        per = max(1, free0 - torch.cuda.mem_get_info(dev)[0])
        fit = torch.tensor([max(1, min(S, 1 + int(torch.cuda.mem_get_info(dev)[0] / 3 // per)))],
                           dtype=torch.int64)
        dist.all_reduce(fit, op=dist.ReduceOp.MIN)
        S = int(fit.item())
        plan_gb = round(per / 1e9, 2)
        while len(pcs) < S:
            add_peer()
        pc = pcs[0]
        n_cap = C.c_uint64()
        from paper_2310_12403_b200.coopbatch import _check
        _check(_lib.load().cb_plan_captured_launches(pc._h, 4, C.byref(n_cap)))

        mb_ = C.c_uint64()
        _lib.load().cb_plan_meta_async(pc._h, None, C.byref(mb_))
        meta_pin = torch.empty((W + K, int(mb_.value)), dtype=torch.uint8).pin_memory()

        def step(i, seeds):
            p_ = pcs[i % S]
            p_.step(seeds, scheds[i])
            if not isinstance(seeds, torch.Tensor):  # e2e: the step's counts come back
                _lib.load().cb_plan_meta_async(p_._h, C.c_void_p(meta_pin[i].data_ptr()), None)
            return 0  # row bytes read from the device after the timed loop
    else:
        eng = CudaEngine(g, pm, rank, L, scfg, max_seeds=b, store=store,
                         comm_device=None if backend == "nccl" else "cpu")
        dc = DistCoop(eng)

        def step(i, seeds):
            dc.sample(seeds, L, scheds[i], keep_blocks=False, records=False)
            return dc.load_inputs(to_host=False).numel()

    for i in range(W):
        step(i, seeds_dev[i])
    lc = C.c_uint64()

    def timed(seeds_of, device_clock=False):
        dist.barrier()
        torch.cuda.synchronize()
        _lib.load().cb_kernel_launches(C.byref(lc))
        l0 = lc.value
        px = args.exchange == "px"
        if px:  # CUDA events on a master stream every plan stream waits on / joins
            master = torch.cuda.current_stream()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(master)
            for p_ in pcs:
                p_.stream.wait_event(e0)
        t = time.perf_counter()
        n_rows = 0
        for i in range(W, W + K):
            n_rows += step(i, seeds_of(i))
        if px:
            for p_ in pcs:
                ev_ = torch.cuda.Event()
                ev_.record(p_.stream)
                master.wait_event(ev_)
            e1.record(master)
            for p_ in pcs:
                p_.finish()
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
        if px and device_clock:
            dt = e0.elapsed_time(e1) / 1e3
        _lib.load().cb_kernel_launches(C.byref(lc))
        launched = lc.value - l0 + (K * n_cap.value if px else 0)
        dist.barrier()
        m = torch.tensor([dt], dtype=torch.float64)
        dist.all_reduce(m, op=dist.ReduceOp.MAX)
        return float(m.item()), n_rows, launched

    clocks = ClockSampler(dev)
    with clocks:
        dt, row_bytes_total, launches = timed(lambda i: seeds_dev[i], device_clock=True)
    if args.exchange == "px":  # the last step's rows, times K
        nr = C.c_uint64()
        row_bytes_total = 0
        for p_ in pcs:  # the last step of every in-flight slot, times K / S
            _lib.load().cb_px_sizes(p_._h, L - 1, C.byref(nr), None)
            row_bytes_total += nr.value * store.row_bytes * K / len(pcs)
    # e2e: host seeds (H2D inside each step), rows end on the device, the
    # step's per-layer counts read back into pinned memory (px) or the split
    # sizes read by the host-orchestrated exchange (a2a)
    e2e_dt, _, _ = timed(lambda i: seeds_host[i])
    if rank != 0:
        dist.destroy_process_group()
        return
    seeds_total = K * b * world
    line = {
        "metric": METRIC, "value": seeds_total / dt, "unit": "seeds/s", "n_gpus": world,
        "steps": K, "warmup": W, "ms_per_step": 1e3 * dt / K, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic (hash-keyed R-MAT, hashed features)",
        "config": {"workload": cfg["workload"],
                   "mode": f"cooperative (P={world}, one part per GPU; " + (
                       "peer-memory exchange: ids OR-ed into owners' bitmaps over CUDA IPC, "
                       "ranks read back; owners stage their requested rows, requesters pull "
                       "them; one device barrier per layer (signal kernel + stream memory "
                       "wait); the whole step is one CUDA graph per rank)"
                       if args.exchange == "px" else
                       f"{backend} all-to-allv per layer + feature all-to-allv)"),
                   "inflight": len(pcs) if args.exchange == "px" else 1,
                   "plan_gb": plan_gb if args.exchange == "px" else None,
                   "timing": ("CUDA events on a master stream joined by the in-flight plans' "
                              "streams around K graph replays, max over ranks"
                              if args.exchange == "px" else
                              "wall clock between barriers + device sync, max over ranks "
                              "(host-orchestrated exchange)"),
                   "graph": {"vertices": cfg["n"], "edges": cfg["m"], "gen_s": round(gen_s, 2)}},
        "feature_gbps": row_bytes_total / dt / 1e9,
        "e2e": {"value": seeds_total / e2e_dt, "unit": "seeds/s", "h2d_bytes_per_step": b * 4,
                "d2h_bytes_per_step": int(mb_.value) if args.exchange == "px" else 8 * (1 + 2 * L)},
        "gpu_launches": launches, "clocks": clocks.summary(),
    }
    print(json.dumps(line), flush=True)
    dist.destroy_process_group()


# -------------------------------------------------------------- our arm ----
def run_ours(args, cfg):
    import torch

    import paper_2310_12403_b200 as cb
    from paper_2310_12403_b200 import _lib
    from paper_2310_12403_b200.seeds import draw_from_pool

    _lib_ = _lib.load()
    rank, world, local = dist_env()
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    torch.cuda.set_device(local)
    dev = local

    kind = {"labor0": cb.SamplerKind.kLabor0, "ns": cb.SamplerKind.kNs,
            "full": cb.SamplerKind.kFull}[cfg["kind"]]
    L = len(cfg["fanouts"])
    b = cfg["batch"]
    t0 = time.time()
    g = cb.Graph.generate_rmat(cfg["n"], cfg["m"], GRAPH_SEED, device=dev)
    gen_s = time.time() - t0
    store = cb.FeatureStore.synth(g, cfg["dim"], FEAT_SEED, cfg["dtype"])
    scfg = cb.SamplerConfig(kind, fanouts=cfg["fanouts"])
    plan = cb.Plan(g, None, L, scfg, b)
    off = np.array([0, b], np.uint64)
    pool = np.arange(cfg["n"], dtype=np.uint32)
    W, K = args.warmup, args.steps
    # per-step seeds of this rank (independent minibatching across ranks)
    tags = [cb.hash_bits(step, [rank]) for step in range(W + K)]
    seeds_host = np.stack([draw_from_pool(pool, b, RUN_SEED, t) for t in tags])
    scheds = [cb.SeedSchedule.make(1, RUN_SEED)]
    for _ in range(W + K):
        scheds.append(cb.schedule_advance(scheds[-1]))

    # one eager batch with overflow-retry sizing, then capture as CUDA graphs
    plan.sample([seeds_host[0]], scheds[0], cb.MODE_INDEP, sync=True)
    plan.capture(off, scheds[0], cb.MODE_INDEP, store)
    stream = torch.cuda.ExternalStream(plan.stream, device=torch.device(f"cuda:{dev}"))
    d_seeds = torch.from_numpy(seeds_host.view(np.int32)).to(f"cuda:{dev}")
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=f"cuda:{dev}")
    clean = torch.empty(64 << 20, dtype=torch.int32, device=f"cuda:{dev}")

    def flush_l2():
        # write 512 MiB (> 126 MB L2), then read 256 MiB so the dirty lines are
        # written back here, outside the timed region
        with torch.cuda.stream(stream):
            flush.zero_()
            clean.sum()
    row_bytes = store.row_bytes

    def step_ptr(i):
        return d_seeds.data_ptr() + i * b * 4

    # S independent minibatches in flight: one plan (captured CUDA graph) and
    # one stream each, step i on plan i % S (a sampler feeding a trainer
    # keeps batches i+1.. in flight while batch i is consumed)
    S = max(1, args.inflight)
    plans, streams = [plan], [stream]
    for _ in range(S - 1):
        p2 = cb.Plan(g, None, L, scfg, b)
        p2.sample([seeds_host[0]], scheds[0], cb.MODE_INDEP, sync=True)
        p2.capture(off, scheds[0], cb.MODE_INDEP, store)
        plans.append(p2)
        streams.append(torch.cuda.ExternalStream(p2.stream, device=torch.device(f"cuda:{dev}")))

    # pinned host buffers of cb_plan_result_async (one per in-flight plan),
    # sized at 4x one warm batch's result
    plans[0].replay(step_ptr(0), scheds[0], True, 3)
    tmp = torch.empty(256 << 20, dtype=torch.uint8).pin_memory()
    plans[0].result_async(tmp.data_ptr(), tmp.numel())
    plans[0].synchronize()
    one = int(tmp.numpy()[:40].view(np.uint64)[3])
    del tmp
    res_cap = max(4 * one, 1 << 20)
    res_bufs = [torch.empty(res_cap, dtype=torch.uint8).pin_memory() for _ in range(S)]
    for j, pl_ in enumerate(plans):  # every plan's pack buffer allocated before timing
        pl_.replay(step_ptr(0), scheds[0], True, 3)
        pl_.result_pack()
        pl_.result_copy(res_bufs[j].data_ptr(), res_cap)
        pl_.synchronize()

    # ---- warmup
    for i in range(W):
        plans[i % S].replay(step_ptr(i), scheds[i], True, 3)
    for pl_ in plans:
        pl_.synchronize()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()

    def run_steps(replay, tail=None):
        """Time K steps round-robin over the S plans: events on a master
        stream that every plan stream waits on / joins."""
        master = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(master)
        for st_ in streams:
            st_.wait_event(e0)
        for i in range(K):
            replay(i)
        if tail:
            tail()
        for st_ in streams:
            ev_ = torch.cuda.Event()
            ev_.record(st_)
            master.wait_event(ev_)
        e1.record(master)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1)

    # ---- latency without a flush: one batch at a time on one stream (inputs
    # are far larger than L2; the code and the plan's metadata stay cached, as
    # in steady-state serving). Run first, so the flushed pass below starts
    # every step cold regardless.
    evu = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(K)]
    for i in range(K):
        evu[i][0].record(stream)
        plan.replay(step_ptr(W + i), scheds[W + i], True, 3)
        evu[i][1].record(stream)
    torch.cuda.synchronize()
    step_ms_unflushed = [e[0].elapsed_time(e[1]) for e in evu]

    # ---- latency: one batch at a time, L2 flushed before every step
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(K)]
    for i in range(K):
        flush_l2()
        ev[i][0].record(stream)
        plan.replay(step_ptr(W + i), scheds[W + i], True, 3)
        ev[i][1].record(stream)
    torch.cuda.synchronize()
    step_ms = [e[0].elapsed_time(e[1]) for e in ev]

    # ---- timed (device-resident inputs): S batches in flight
    clocks = ClockSampler(dev)
    with clocks:
        total_ms = run_steps(lambda i: plans[i % S].replay(step_ptr(W + i), scheds[W + i],
                                                           True, 3))
    for pl_ in plans:
        pl_.synchronize()  # raises on capacity overflow
    if world > 1:
        torch.distributed.barrier()
    sizes = [plan.layer_sizes(0, l) for l in range(L)]
    rows_last = sizes[-1]["n_src"]
    if world > 1:
        t = torch.tensor([total_ms], device=f"cuda:{dev}")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_ms = float(t.item())

    # ---- e2e through the C-ABI with host buffers: every step the seeds (+
    # variate keys) go H2D from pinned memory inside the replay, and the whole
    # batch result -- every layer's block and the gathered rows -- is written
    # into a pinned host buffer by cb_plan_result_async (one kernel, counts
    # read on the device); all S streams joined at the end, wall clock
    pinned = torch.from_numpy(seeds_host.view(np.int32)).pin_memory()
    res_cap_used = res_cap

    # the result of batch i leaves by the copy engines (cb_plan_result_copy):
    # issued just before plan i % S takes batch i + S, so the host waits on
    # the oldest batch while S - 1 newer ones keep the device busy
    host_t = {"copy": 0.0, "replay": 0.0}

    def e2e_step(i):
        t_ = time.perf_counter()
        if i >= S:
            plans[i % S].result_copy(res_bufs[i % S].data_ptr(), res_cap_used)
        t1_ = time.perf_counter()
        plans[i % S].replay(pinned.data_ptr() + (W + i) * b * 4, scheds[W + i], False, 3)
        plans[i % S].result_pack()  # packed on the device right behind the batch
        host_t["copy"] += t1_ - t_
        host_t["replay"] += time.perf_counter() - t1_

    def e2e_tail():
        for i in range(max(0, K - S), K):
            plans[i % S].result_copy(res_bufs[i % S].data_ptr(), res_cap_used)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    te = time.perf_counter()
    e2e_ms = run_steps(e2e_step, e2e_tail)
    e2e_s = time.perf_counter() - te
    if world > 1:
        t = torch.tensor([e2e_s], device=f"cuda:{dev}")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_s = float(t.item())
    res_bytes = []
    for j in range(min(S, K)):  # the last result of every slot
        hd = res_bufs[j].numpy()[:40].view(np.uint64)
        assert int(hd[4]) == 0, "e2e result buffer truncated"
        res_bytes.append(int(hd[3]))
    last = cb.parse_result(res_bufs[(K - 1) % S].numpy())
    assert last["blocks"][L - 1]["src"].size > 0, "e2e batch result read back empty"
    # ---- e2e with the result left on the device (only the per-layer counts
    # read back): the sampler-feeding-a-GPU-trainer case
    mb = C.c_uint64()
    _lib_.cb_plan_meta_async(plan._h, None, C.byref(mb))
    meta_h = torch.empty((K, int(mb.value)), dtype=torch.uint8).pin_memory()

    def e2e_dev_step(i):
        plans[i % S].replay(pinned.data_ptr() + (W + i) * b * 4, scheds[W + i], False, 3)
        _lib_.cb_plan_meta_async(plans[i % S]._h, C.c_void_p(meta_h[i].data_ptr()), None)
    torch.cuda.synchronize()
    td = time.perf_counter()
    run_steps(e2e_dev_step)
    e2e_dev_s = time.perf_counter() - td
    if world > 1:
        t = torch.tensor([e2e_dev_s], device=f"cuda:{dev}")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_dev_s = float(t.item())
    launches_per_step = plan.captured_launches(3)  # the replayed sample + gather graph
    # per-launch device times of one batch (step W's seeds and schedule)
    # inside the CUDA graph (event-record nodes on the plan stream), L2
    # flushed before each of R replays, averaged per launch
    prof_runs = []
    for _ in range(5):
        flush_l2()
        prof_runs.append(plan.graph_profile(step_ptr(W), scheds[W]))
    prof_ms = [float(x) for x in np.mean(np.array(prof_runs), axis=0)]
    prof_sizes = [plan.layer_sizes(0, l) for l in range(L)]
    rows_last = prof_sizes[-1]["n_src"]
    # the gather alone on that batch, events on its stream, L2 flushed before
    # every launch
    gev = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(K)]
    for i in range(K):
        flush_l2()
        gev[i][0].record(stream)
        plan.gather(store)  # one gather_kernel launch on the plan stream
        gev[i][1].record(stream)
    torch.cuda.synchronize()
    gath_ms = [e[0].elapsed_time(e[1]) for e in gev]
    samp_ms = [s_ - float(np.mean(gath_ms)) for s_ in step_ms]
    if rank != 0:
        return
    traffic = ({"error": "skipped (--no-traffic)"} if args.no_traffic else
               ncu_traffic(args.config, W))
    seeds_total = K * b * world
    value = seeds_total / (total_ms / 1000.0)
    peak, peak_kind = peaks()
    # dominant kernel: the gather (one launch per step)
    gather_bytes = rows_last * (2 * row_bytes + 4)
    gather_avg_s = float(np.mean(gath_ms)) / 1000.0
    achieved = gather_bytes / gather_avg_s / 1e9
    feat_gbps = rows_last * row_bytes / gather_avg_s / 1e9
    line = {
        "metric": METRIC, "value": value, "unit": "seeds/s", "n_gpus": world, "steps": K,
        "warmup": W, "ms_per_step": total_ms / K, "higher_is_better": True, "scaling": "weak",
        "latency_ms_per_step": float(np.mean(step_ms)),
        "latency_unflushed_ms_per_step": float(np.mean(step_ms_unflushed)),
        "vs_baseline": None, "dtype": "u32", "data": "synthetic (hash-keyed R-MAT, hashed "
        "features; random-init equivalent)",
        "config": {"workload": cfg["workload"], "mode": "indep (P=1 per GPU)",
                   "inflight": S,
                   "l2": (f"not flushed: inputs larger than L2 (CSR {g.num_edges() * 4 / 1e9:.2f} GB"
                          f" + feature table {cfg['n'] * row_bytes / 1e9:.2f} GB vs 126 MB); "
                          f"{S} minibatches in flight on {S} streams. latency_ms_per_step: one "
                          "batch at a time, L2 flushed before every step (512 MiB write + "
                          "256 MiB read, untimed); latency_unflushed_ms_per_step: one batch at "
                          "a time, no flush (inputs larger than L2)") if S > 1 else
                         "flushed before every step (512 MiB write + 256 MiB read, untimed)",
                   "graph": {"vertices": cfg["n"], "edges": cfg["m"],
                             "max_degree": g.max_degree, "gen_s": round(gen_s, 2)},
                   "cuda_graphs": True},
        "feature_gbps": feat_gbps,
        "stage_ms": {"sample_dedup": float(np.mean(samp_ms)), "gather": float(np.mean(gath_ms)),
                     "note": "gather timed alone (one launch, events on its stream); sample = step - gather"},
        "e2e": {"value": seeds_total / e2e_s, "unit": "seeds/s",
                "h2d_bytes_per_step": b * 4 + 40,
                "d2h_bytes_per_step": int(np.mean(res_bytes)),
                "result": "every layer's dst/src/edges/dst_pos + the gathered rows, copied "
                          "into pinned host memory by the copy engines each step "
                          "(cb_plan_result_copy, S batches in flight)",
                "device_ms": e2e_ms,
                "host_ms": {k_: round(1e3 * v_, 2) for k_, v_ in host_t.items()}},
        "e2e_device_result": {"value": seeds_total / e2e_dev_s, "unit": "seeds/s",
                              "h2d_bytes_per_step": b * 4 + 40,
                              "d2h_bytes_per_step": int(mb.value),
                              "result": "left in HBM for a GPU consumer; per-layer counts "
                                        "read back (cb_plan_meta_async)"},
        "roofline": mark_roofline(prof_ms, prof_sizes, L, scfg, peak, peak_kind, traffic),
        "roofline_gather": {
            "bound": "hbm",
            "kernel": "gather_kernel<V,U> (16/8/4/2-byte vectors by row size; U = 3 for "
                      "16-byte, else 4)",
            "achieved": achieved, "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
            "frac": achieved / peak, "traffic": traffic.get("gather"),
            "bytes_per_launch": gather_bytes,
            "per_unit": "per input row: owner row read + requester row write + 4 B id",
            "ms": float(np.mean(gath_ms)), "share_of_batch": prof_ms[-1] / sum(prof_ms)},
        "traffic_probe": traffic,
        "gpu_launches": launches_per_step * K,
        "kernel_ms_graph": [round(x, 4) for x in prof_ms],
        "evidence": {"per_layer": sizes,
                     "sampled_vertices_per_seed": rows_last / b,
                     "feature_bytes_per_step": rows_last * row_bytes},
        "clocks": clocks.summary(),
    }
    plans.clear()  # the evidence runs make their own plans
    streams.clear()
    plan = p2 = None  # noqa: F841
    if world == 1 and not args.no_evidence:
        line["evidence"]["concavity"] = concavity_evidence(cb, g, scfg, L, b, row_bytes, dev)
        line["evidence"]["kappa"] = kappa_evidence(cb, dev)
        other = "c2" if args.config == "c4" else "c4"
        line["evidence"]["products_c2" if other == "c2" else "papers100m"] = \
            scale_evidence(cb, dev, other)
        line["evidence"]["mag240m_batch_sweep"] = batch_sweep_evidence(cb, dev)
        line["evidence"]["work_curves"] = work_curve_evidence(cb, dev, not args.no_cpu_baseline)
        line["evidence"]["dropin_e2e_c2"] = dropin_evidence()
    if world == 1 and not args.no_cpu_baseline:
        try:
            from oracle import oracle as O
            indptr, indices = g.download()
            csr = O.CSR(indptr, indices)
            v, cores, desc, _ = cpu_reference_leg(cfg, csr, args.cpu_budget)
            line["cpu_baseline"] = {"value": v, "unit": "seeds/s", "cores": cores,
                                    "kind": "reference", "sample": desc}
        except Exception as e:  # report, never fake
            line["cpu_baseline"] = {"value": None, "error": str(e)[:200]}
    print(json.dumps(line), flush=True)
    if args.csv_dir:
        write_reports(args, cfg)


def write_reports(args, cfg):
    """The reference CLI's CSV reports (reports.py) of the evidence runs."""
    from paper_2310_12403_b200 import reports as R
    os.makedirs(args.csv_dir, exist_ok=True)
    base = {"config": args.config, "layers": len(cfg["fanouts"]),
            "fanout": "/".join(map(str, cfg["fanouts"])), "batch": cfg["batch"],
            "sampler": cfg["kind"], "graph_seed": GRAPH_SEED, "run_seed": RUN_SEED}
    for kappa, rows in CSV_ROWS.get("cache", []):
        R.write_csv(os.path.join(args.csv_dir, f"cache_c3_kappa{kappa or 'inf'}.csv"),
                    {**base, "config": "c3", "kappa": kappa or "inf", "mode": "smoothed"},
                    R.CACHE_COLUMNS, rows)
    if CSV_ROWS.get("curve"):
        c5 = CONFIGS["c5"]
        R.write_csv(os.path.join(args.csv_dir, "curve_c5.csv"),
                    {**base, "config": "c5", "layers": len(c5["fanouts"]),
                     "fanout": "/".join(map(str, c5["fanouts"])), "batch": "sweep"},
                    R.curve_columns(len(c5["fanouts"])), CSV_ROWS["curve"])
    by_sampler = {}
    for name, b, mean, se, wps, _sew in CSV_ROWS.get("work_curve", []):
        by_sampler.setdefault(name, []).append((b, mean, se, wps))
    for name, rows in by_sampler.items():
        R.write_csv(os.path.join(args.csv_dir, f"curve_c1_{name}.csv"),
                    {**base, "config": "c1", "sampler": name, "layers": 3, "trials": 50,
                     "batch": "64..8192"}, R.curve_columns(3), rows)
    run = []
    for tag, metrics in CSV_ROWS.get("run", []):
        run.extend(R.run_rows(0, tag, metrics))
    if run:
        R.write_csv(os.path.join(args.csv_dir, "run_concavity.csv"), base, R.RUN_COLUMNS, run)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="c4", choices=sorted(CONFIGS))
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-evidence", action="store_true")
    ap.add_argument("--csv-dir", default="", help="also write the evidence as CLI-format CSVs")
    ap.add_argument("--probe", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--probe-step", type=int, default=0, help=argparse.SUPPRESS)
    ap.add_argument("--no-traffic", action="store_true",
                    help="skip the in-run ncu DRAM-traffic measurement")
    ap.add_argument("--inflight", type=int, default=8,
                    help="independent minibatches in flight per GPU (streams); 1 = one at a time")
    ap.add_argument("--mode", choices=["coop", "indep"], default="coop",
                    help="N>1: cooperative minibatching (one part per GPU) or independent")
    ap.add_argument("--exchange", choices=["px", "a2a"], default="px",
                    help="N>1 coop: peer-memory exchange (cb_px_*) or all-to-allv (DistCoop)")
    ap.add_argument("--coop-n1", action="store_true",
                    help="run the cooperative (peer-exchange) step even at N=1 (diagnostics)")
    ap.add_argument("--dist-backend", choices=["nccl", "gloo"], default="nccl",
                    help="gloo: ranks share cuda:0 with CPU-staged exchanges (testing)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    cfg = CONFIGS[args.config]
    rank, world, _ = dist_env()
    if args.probe:
        run_probe(args, cfg)
        return
    if args.impl == "reference":
        run_reference(args, cfg)
    elif (world > 1 or args.coop_n1) and args.mode == "coop":
        run_ours_coop(args, cfg)
        return
    else:
        run_ours(args, cfg)
    if world > 1 and args.impl == "ours":
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
