"""Loader for tests/golden/golden.npz (written by tests/golden/make_golden.py)."""

import functools
import json
import os

import numpy as np

PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden.npz")


@functools.lru_cache(maxsize=1)
def _load():
    z = np.load(PATH)
    meta = json.loads(str(z["meta"]))
    arrays = {k: z[k] for k in z.files if k != "meta"}
    return arrays, {m["name"]: m for m in meta}


def bits_to_f64(bits):
    b = np.asarray(bits, dtype=np.uint16).astype(np.uint32) << 16
    return b.view(np.float32).astype(np.float64)


def case_names():
    return list(_load()[1])


def case(name):
    """Returns (meta dict, q, k, v as float64 (exact bf16 values), out f32, lse f64)."""
    arrays, meta = _load()
    m = meta[name]
    q, k, v = (bits_to_f64(arrays[m[f"in_{t}"]]) for t in "qkv")
    return m, q, k, v, arrays[f"{name}/out"], arrays[f"{name}/lse"]


def case_bits(name):
    arrays, meta = _load()
    m = meta[name]
    return tuple(arrays[m[f"in_{t}"]] for t in "qkv")


def case_stab(name):
    """Reference stabilization positions per row (None if the case has no StateTrace)."""
    arrays, _ = _load()
    return arrays.get(f"{name}/stab")
