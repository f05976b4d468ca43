"""Summarise one GPU round (gpurun_out/<tag>) into profiles/: the ncu launch
list of the bench command (per-launch gpu__time_duration, clock-control none),
key metrics of each `ncu --set full` capture, and profiles/ncu_traffic.json
(per-launch DRAM bytes of the roofline kernel, read by bench.py).

  python tools/summarize_profiles.py gpurun_out/r01c r01 [dim]
"""
import csv
import io
import json
import os
import shutil
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "lts__t_sector_hit_rate.pct",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__occupancy_limit_registers", "gpc__cycles_elapsed.max"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u = rows[0], rows[1]
    res = []
    for d in rows[2:]:
        m = {"kernel": d[h.index("Kernel Name")]}
        for k in KEYS:
            if k in h:
                i = h.index(k)
                m[k] = (d[i], u[i])
        res.append(m)
    return res


def to_bytes(v):
    return float(v[0].replace(",", "")) * SCALE.get(v[1], 1)


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    return data


def main():
    src, tag = sys.argv[1], sys.argv[2]
    dim = int(sys.argv[3]) if len(sys.argv) > 3 else 100
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    dst = os.path.join(root, "profiles")
    os.makedirs(dst, exist_ok=True)
    md = [f"# {tag}: ncu summary of `python bench.py` (N=1)\n"]
    if os.path.exists(os.path.join(src, "bench.json")):
        b = json.loads(open(os.path.join(src, "bench.json")).read().strip().splitlines()[-1])
        shutil.copy(os.path.join(src, "bench.json"), os.path.join(dst, f"{tag}_bench.json"))
        md.append(f"workload: {b['config'].get('workload', '?')}\n")
        rf = b["roofline"]
        md.append(f"bench: value {b['value']:.0f} seeds/s, {b['ms_per_step']*1e3:.1f} us/step, "
                  f"e2e {b['e2e']['value']:.0f} seeds/s; roofline ({rf.get('kernel', '?')}) frac "
                  f"{rf['frac']:.3f} ({rf['achieved']:.0f} GB/s)")
        if "roofline_gather" in b:
            rg = b["roofline_gather"]
            md.append(f"; gather frac {rg['frac']:.3f} ({rg['achieved']:.0f} GB/s)")
        md.append("\n")
    lp = os.path.join(src, "launches.csv")
    if os.path.exists(lp):
        data = launches(lp)
        shutil.copy(lp, os.path.join(dst, f"{tag}_launches.csv"))
        # last step's launches = everything after the last batch_begin
        last = max(i for i, d in enumerate(data) if "batch_begin" in d["Kernel Name"])
        # the eager gather timing loop follows the graph replays: take the
        # last complete batch (batch_begin .. gather)
        starts = [i for i, d in enumerate(data) if "batch_begin" in d["Kernel Name"]]
        segs = [data[a:b] for a, b in zip(starts, starts[1:] + [len(data)])]
        # an indep P=1 batch: begin, L x (frontier, mark, post), relabel, gather
        full = [sg for sg in segs if any("gather" in d["Kernel Name"] for d in sg)
                and sum("frontier" in d["Kernel Name"] for d in sg) == 3
                and sum("relabel" in d["Kernel Name"] for d in sg) == 1]
        step = full[-1] if full else data[last:]
        # keep the batch and its own gather only
        gi = max(i for i, d in enumerate(step) if "gather" in d["Kernel Name"]) \
            if full else len(step) - 1
        step = step[:gi + 1]
        tot = sum(float(d["Metric Value"].replace(",", "")) for d in step)
        md.append("\n## One batch, per launch (ns, cold-cache serialised)\n\n| # | kernel | grid | ns | share |\n|---|---|---|---|---|")
        for i, d in enumerate(step):
            ns = float(d["Metric Value"].replace(",", ""))
            md.append(f"| {i} | `{d['Kernel Name'][:60]}` | {d['Grid Size']} | {ns:.0f} | "
                      f"{ns / tot:.1%} |")
        md.append(f"\nbatch total {tot/1e3:.1f} us over {len(step)} launches\n")
    traffic = {}
    for rep in sorted(f for f in os.listdir(src) if f.endswith(".ncu-rep")):
        for m in raw(os.path.join(src, rep)):
            md.append(f"\n## `{m['kernel'][:90]}` ({rep}, --set full)\n")
            for k in KEYS:
                if k in m:
                    md.append(f"- {k}: {m[k][0]} {m[k][1]}")
            if "gather" in m["kernel"]:
                traffic["gather"] = {
                    "dram_bytes": to_bytes(m["dram__bytes_read.sum"]) +
                    to_bytes(m["dram__bytes_write.sum"]), "dim": dim, "source": f"{tag}/{rep}"}
        shutil.copy(os.path.join(src, rep), os.path.join(dst, f"{tag}_{rep}"))
    if traffic:
        json.dump(traffic, open(os.path.join(dst, "ncu_traffic.json"), "w"), indent=1)
    open(os.path.join(dst, f"{tag}_summary.md"), "w").write("\n".join(md) + "\n")


if __name__ == "__main__":
    main()
