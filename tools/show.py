import json, sys, glob
for f in sorted(glob.glob(sys.argv[1] + "/bench*.json")):
    try:
        b = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, round(b["ms_per_step"] * 1000, 1), "us  e2e", round(b["e2e"]["value"]),
              "frac", round(b["roofline"]["frac"], 3), b.get("kernel_ms_graph"))
    except Exception as e:
        print(f, "ERR", e)
