"""CSV reports in the reference CLI's formats (cli.cpp:74-99): every file
starts with `# key=value` lines of the resolved configuration and is written
atomically (temp file, then rename). Column sets follow the CLI's:
  run      step,mode,pe,layer,s_l,s_tilde_l,e_l,comm_vertices,feat_bytes,loss (cli.cpp:208)
  curve    batch_size,mean_s<L>,se_s<L>,work_per_seed                     (cli.cpp:184-188)
  cache    step,miss_rate,s_l,bytes                                       (cli.cpp:256)
  partition vertex,part                                                   (cli.cpp:153-162)
Floating-point fields are printed like the CLI's std::ostream defaults (six
significant digits, %g).
"""
from __future__ import annotations

import os

RUN_COLUMNS = ["step", "mode", "pe", "layer", "s_l", "s_tilde_l", "e_l", "comm_vertices",
               "feat_bytes", "loss"]
CACHE_COLUMNS = ["step", "miss_rate", "s_l", "bytes"]
PARTITION_COLUMNS = ["vertex", "part"]


def curve_columns(layers: int) -> list[str]:
    """cli.cpp:184-185: the curve header names the layer count."""
    return ["batch_size", f"mean_s{layers}", f"se_s{layers}", "work_per_seed"]


CURVE_COLUMNS = curve_columns(3)


def write_csv(path: str, config: dict, columns: list[str], rows) -> None:
    tmp = path + ".tmp"
    with open(tmp, "w") as f:
        for k, v in config.items():
            f.write(f"# {k}={v}\n")
        f.write(",".join(columns) + "\n")
        for r in rows:
            f.write(",".join(_fmt(x) for x in r) + "\n")
    os.replace(tmp, path)


def _fmt(x) -> str:
    if isinstance(x, float):
        return f"{x:g}"  # std::ostream << double (precision 6)
    return str(x)


def curve_rows(curve):
    """Rows of the `curve` report from analysis.WorkCurve (cli.cpp:186-188)."""
    for p in curve.points:
        yield (p.batch_size, p.mean_sl, p.se_sl, p.work_per_seed)


def partition_rows(owner):
    """Rows of the `partition` report: one (vertex, part) per vertex (cli.cpp:158-161)."""
    for v, p in enumerate(owner.tolist() if hasattr(owner, "tolist") else owner):
        yield (v, p)


def run_rows(step: int, mode: str, metrics, loss: float = 0.0):
    """Rows of the `run` report from step_metrics (LayerMetrics per PE)."""
    for p, pe in enumerate(metrics):
        for l, m in enumerate(pe.layers):
            yield (step, mode, p, l, m.s_l, m.s_tilde_l, m.e_l, m.comm_vertices, pe.feat_bytes,
                   loss)
