"""Shared test helpers: rebuild golden-case inputs with the package's own
(bit-identical, hash-pinned) host generators."""

import json

import numpy as np

from paper_2602_13140_b200.modelparams import ModelConfig, init_params
from paper_2602_13140_b200.w16 import quantize_model

_QCACHE = {}


def params_for(case) -> object:
    cfg = ModelConfig(**json.loads(str(case["cfg"])))
    seed = int(case["pseed"])
    p = init_params(cfg, seed)
    if case["pos"].dtype == np.float64:
        p = p.astype(np.float64)
    if bool(case.get("quant", False)):
        key = (str(case["cfg"]), seed)
        if key not in _QCACHE:
            _QCACHE[key] = quantize_model(p, seed=0)
        p = _QCACHE[key]
    return p


def quantized(params):
    """quantize_model(params, seed=0), cached per params object."""
    key = ("obj", id(params))
    if key not in _QCACHE or _QCACHE[key][0] is not params:
        _QCACHE[key] = (params, quantize_model(params, seed=0))
    return _QCACHE[key][1]


def rel_rmse(f, ref):
    return float(np.sqrt(np.mean((f - ref) ** 2)) / np.sqrt(np.mean(ref ** 2)))
