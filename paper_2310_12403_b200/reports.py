"""CSV reports in the reference CLI's formats (cli.cpp:74-99): every file
starts with `# key=value` lines of the resolved configuration and is written
atomically (temp file, then rename). Column sets follow the CLI's:
  run      step,mode,pe,layer,s_l,s_tilde_l,e_l,comm_vertices,feat_bytes,loss (cli.cpp:208)
  curve    batch_size,mean_sL,se_sL,work_per_seed                         (cli.cpp:184-185)
  cache    step,miss_rate,s_l,bytes                                       (cli.cpp:256)
"""
from __future__ import annotations

import os

RUN_COLUMNS = ["step", "mode", "pe", "layer", "s_l", "s_tilde_l", "e_l", "comm_vertices",
               "feat_bytes", "loss"]
CURVE_COLUMNS = ["batch_size", "mean_sL", "se_sL", "work_per_seed"]
CACHE_COLUMNS = ["step", "miss_rate", "s_l", "bytes"]


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
        return repr(x)
    return str(x)


def run_rows(step: int, mode: str, metrics, loss: float = 0.0):
    """Rows of the `run` report from step_metrics (LayerMetrics per PE)."""
    for p, pe in enumerate(metrics):
        for l, m in enumerate(pe.layers):
            yield (step, mode, p, l, m.s_l, m.s_tilde_l, m.e_l, m.comm_vertices, pe.feat_bytes,
                   loss)
