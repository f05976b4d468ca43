"""Host mirror of the reference's GCN training step (coop.hpp:105-185):
``GcnModel`` (weights on the device), ``coop_train_step`` and
``indep_train_step`` over libcoopbatch_b200 (csrc/train.cu). The sampling,
exchange records and feature rows of the step come from the same device
plan as coop_sample / load_inputs; the forward/backward passes run in FP64
in the reference's accumulation order."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .coopbatch import (MODE_COOP, MODE_INDEP, FeatureStore, Graph, InputError, PartitionMap,
                        SamplerConfig, SeedSchedule, _check, _plan_for, _ptr)


class GcnModel:  # coop.hpp:126-135
    def __init__(self, handle, num_layers: int, device: int):
        self._h, self.num_layers, self.device = handle, num_layers, device

    @classmethod
    def init(cls, in_dim: int, hidden: int, num_classes: int, num_layers: int, seed: int,
             device: int = 0) -> "GcnModel":
        """GcnModel::init (coop.cpp:334-357)."""
        if num_layers < 1:
            raise InputError("GcnModel: num_layers must be >= 1")
        h = C.c_void_p()
        _check(_lib.load().cb_gcn_model_init(device, in_dim, hidden, num_classes, num_layers,
                                             seed, C.byref(h)))
        return cls(h, num_layers, device)

    def shape(self, layer: int) -> tuple[int, int]:
        r, c = C.c_uint64(), C.c_uint64()
        _check(_lib.load().cb_gcn_model_weights(self._h, layer, None, 0, C.byref(r), C.byref(c)))
        return r.value, c.value

    def weights(self, layer: int) -> np.ndarray:
        r, c = self.shape(layer)
        w = np.zeros((r, c), np.float64)
        _check(_lib.load().cb_gcn_model_weights(self._h, layer, _ptr(w), 0, None, None))
        return w

    def set_weights(self, layer: int, w: np.ndarray):
        r, c = self.shape(layer)
        w = np.ascontiguousarray(w, dtype=np.float64)
        if w.shape != (r, c):
            raise InputError("GcnModel: weight shape mismatch")
        _check(_lib.load().cb_gcn_model_weights(self._h, layer, _ptr(w), 1, None, None))

    def __del__(self):
        try:
            if getattr(self, "_h", None):
                _lib.load().cb_gcn_model_destroy(self._h)
                self._h = None
        except Exception:  # interpreter shutdown
            pass


@dataclass
class TrainStepResult:  # coop.hpp:175-179
    loss: float = 0.0
    grad_w: list[np.ndarray] = field(default_factory=list)


def _step(plan, store: FeatureStore, num_classes: int, model: GcnModel) -> TrainStepResult:
    shapes = [model.shape(l) for l in range(model.num_layers)]
    gw = np.zeros(sum(r * c for r, c in shapes), np.float64)
    loss = C.c_double()
    _check(_lib.load().cb_train_step(plan._h, store._h, num_classes, model._h, C.byref(loss),
                                     _ptr(gw)))
    out, o = [], 0
    for r, c in shapes:
        out.append(gw[o:o + r * c].reshape(r, c).copy())
        o += r * c
    return TrainStepResult(loss.value, out)


def coop_train_step(g: Graph, pm: PartitionMap, per_pe_seeds, num_layers: int,
                    cfg: SamplerConfig, schedule: SeedSchedule, model: GcnModel,
                    store: FeatureStore, num_classes: int) -> TrainStepResult:
    """coop.cpp:438-556: cooperative sample, owner-side feature load +
    all_to_all_forward, GCN forward with hidden-row exchanges, softmax CE on
    the seeds, backward with all_to_all_reverse_sum, gradients summed over
    parts. `store` is an f64 table sharded by `pm` (FeatureStore.synth(...,
    "f64", pm)); labels are hash(seed,{10,v}) mod num_classes."""
    if len(per_pe_seeds) != pm.num_parts:
        raise InputError("coop_sample: seed lists must match the partition count")
    n = max((len(s) for s in per_pe_seeds), default=1)
    pl = _plan_for(g, pm, num_layers, cfg, n)
    pl.sample(per_pe_seeds, schedule, MODE_COOP)
    return _step(pl, store, num_classes, model)


def indep_train_step(g: Graph, per_pe_seeds, num_layers: int, cfg: SamplerConfig,
                     schedule: SeedSchedule, model: GcnModel, store: FeatureStore,
                     num_classes: int) -> TrainStepResult:
    """coop.cpp:560-610: every part samples and trains on its own seeds;
    losses and gradients summed over parts. One plan holds all parts."""
    P = len(per_pe_seeds)
    if P == 0:
        raise InputError("indep_train_step: no parts")
    n = max((len(s) for s in per_pe_seeds), default=1)
    # a P-part plan in independent mode (the partition only sets the part count)
    pl = _plan_for(g, None if P == 1 else _dummy_pm(g, P), num_layers, cfg, n)
    pl.sample(per_pe_seeds, schedule, MODE_INDEP)
    return _step(pl, store, num_classes, model)


_pm_cache: dict = {}


def _dummy_pm(g: Graph, P: int):
    from .coopbatch import partition_random
    key = (id(g), P)
    if key not in _pm_cache:
        _pm_cache[key] = partition_random(g, P, 0)
    return _pm_cache[key]
