"""How much of each LABOR layer's scan space lies in full single-record tiles
(labor_mark phase A) at a bench config. Not part of the product.

  python tools/pure_share.py [c4]
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_2310_12403_b200 as cb  # noqa: E402
from paper_2310_12403_b200.seeds import draw_from_pool  # noqa: E402

TILE = 1024


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c4"
    cfg = bench.CONFIGS[name]
    g = cb.Graph.generate_rmat(cfg["n"], cfg["m"], bench.GRAPH_SEED, device=0)
    indptr, _ = g.download()
    deg = np.diff(indptr).astype(np.int64)
    seeds = draw_from_pool(np.arange(cfg["n"], dtype=np.uint32), cfg["batch"], bench.RUN_SEED, 0)
    sc = cb.SamplerConfig(cb.SamplerKind.kLabor0, cfg["fanouts"][0])
    L = len(cfg["fanouts"])
    st = cb.expand(g, seeds, L, sc, cb.SeedSchedule.make(1, bench.RUN_SEED))
    for l, b in enumerate(st.blocks):
        d = deg[b.dst_vertices]
        d = d[d > 0]
        pre = np.concatenate([[0], np.cumsum(d)])
        total = int(pre[-1])
        nt = total // TILE
        # tile t is pure iff one record covers [t*TILE, (t+1)*TILE)
        starts = np.arange(nt, dtype=np.int64) * TILE
        rec = np.searchsorted(pre, starts, side="right") - 1
        pure = pre[rec + 1] >= starts + TILE
        big = d >= TILE
        print(f"layer {l}: dst {len(b.dst_vertices)} scan {total} tiles {nt} pure {pure.sum()} "
              f"({pure.sum() * TILE / max(total, 1):.3f} of positions); records d>=1024: "
              f"{big.sum()} holding {d[big].sum() / max(total, 1):.3f}; max d {d.max() if len(d) else 0}")


if __name__ == "__main__":
    main()
