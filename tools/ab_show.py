"""Summarise tools/ab.sh output: per variant, ms/step and per-launch graph times."""
import glob
import json
import sys
from collections import defaultdict

d = defaultdict(list)
for f in sorted(glob.glob(f"gpurun_out/{sys.argv[1]}/*.json")):
    name = f.split("/")[-1].rsplit("_", 1)[0]
    try:
        line = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception:
        print("bad", f)
        continue
    d[name].append(line)
for k, ls in d.items():
    ms = [x["ms_per_step"] * 1e3 for x in ls]
    lat = [x["latency_ms_per_step"] * 1e3 for x in ls]
    kg = [round(sum(v) / len(v) * 1e3, 1) for v in zip(*[x["kernel_ms_graph"] for x in ls])]
    print(f"{k:8s} us/step {['%.1f' % m for m in ms]} lat {['%.1f' % m for m in lat]} kernels {kg}")
