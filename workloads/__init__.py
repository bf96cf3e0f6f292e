"""Seeded synthetic inputs shared by the oracle, the tests and bench.py.

This module holds NO arithmetic of the method (no fusion rule, no scaling,
no reduction, no chunking).  It only says *which* tensors a synthetic
gradient set has and *what values* rank r holds, so that the CPU oracle
(``oracle/``) and the CUDA path (``paper_1802_05799_b200``) can be fed the
same bytes without sharing code (task rule ③).

Value representation (numpy):
  * ``"f32"``  -> ``np.float32``
  * ``"bf16"`` -> ``np.uint16`` holding bfloat16 bit patterns
  * ``"i32"``  -> ``np.int32``
  * ``"i64"``  -> ``np.int64``

Recipes:
  * ``normal``:     x_{r,k} = sigma_k * N(0,1), sigma_k = 2^-(k mod 16), numpy
                    PCG64 seeded ``seed + 7919*r + k``; bf16 values are the
                    fp32 draw rounded by ml_dtypes (a library cast).
  * ``ones``:       all 1.
  * ``rank_index``: x_{r,k}[i] = r.
  * ``small_int``:  uniform integers in [-8, 8] (exact in every dtype).
  * ``int_uniform``: uniform integers in [-2^20, 2^20].
  * ``specials``:   normal draws with +-0, +-inf, NaN, subnormals, +-max
                    finite sprinkled in.
"""
from __future__ import annotations

import json
import pathlib

import numpy as np

try:  # ml_dtypes ships with the image; it is only used to make bf16 inputs
    import ml_dtypes as _mld
except ImportError:  # pragma: no cover
    _mld = None

SEED = 180205799  # arXiv id, SURVEY.md §8d
_SHAPES = json.loads((pathlib.Path(__file__).with_name("model_shapes.json")).read_text())

NP_DTYPE = {"f32": np.float32, "bf16": np.uint16, "i32": np.int32, "i64": np.int64}
ELEM_SIZE = {"f32": 4, "bf16": 2, "i32": 4, "i64": 8}


def model_names():
    return sorted(_SHAPES)


def gradient_set(model: str):
    """Parameter (name, numel) list of a torchvision model in SUBMISSION order.

    Submission order is the reverse of registration order, i.e. the order
    backprop makes gradients ready ("Determine which tensors are
    ready").
    """
    out = []
    for name, shape in reversed(_SHAPES[model]):
        n = 1
        for d in shape:
            n *= d
        out.append((name, n))
    return out


def _to_bf16_bits(x32: np.ndarray) -> np.ndarray:
    if _mld is None:  # pragma: no cover
        raise RuntimeError("ml_dtypes is required to generate bf16 inputs")
    return x32.astype(_mld.bfloat16).view(np.uint16)


def _float_values(rng, count, k, kind):
    if kind == "normal":
        sigma = np.float32(2.0 ** -(k % 16))
        return (rng.standard_normal(count, dtype=np.float32) * sigma).astype(np.float32)
    if kind == "specials":
        x = rng.standard_normal(count, dtype=np.float32)
        if count:
            specials = np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 1e-40, -1e-40,
                                 3.0e38, -3.0e38, 1e-45], dtype=np.float32)
            idx = rng.integers(0, count, size=max(1, count // 50))
            x[idx] = specials[rng.integers(0, len(specials), size=len(idx))]
        return x
    raise ValueError(kind)


def rank_tensor(count: int, dtype: str, rank: int, k: int, kind: str = "normal",
                seed: int = SEED) -> np.ndarray:
    """Values of tensor k on rank ``rank`` (flat, numpy, see module doc)."""
    rng = np.random.Generator(np.random.PCG64(seed + 7919 * rank + k))
    if kind == "ones":
        v = np.ones(count, dtype=np.float64)
    elif kind == "rank_index":
        v = np.full(count, float(rank))
    elif kind == "small_int":
        v = rng.integers(-8, 9, size=count).astype(np.float64)
    elif kind == "int_uniform":
        v = rng.integers(-(1 << 20), (1 << 20) + 1, size=count).astype(np.float64)
    elif kind in ("normal", "specials"):
        if dtype in ("i32", "i64"):
            raise ValueError("float recipe for an integer dtype")
        x32 = _float_values(rng, count, k, kind)
        return x32 if dtype == "f32" else _to_bf16_bits(x32)
    else:
        raise ValueError(kind)
    if dtype == "f32":
        return v.astype(np.float32)
    if dtype == "bf16":
        return _to_bf16_bits(v.astype(np.float32))
    return v.astype(NP_DTYPE[dtype])


def rank_tensors(counts, dtype, rank, kind="normal", seed=SEED):
    return [rank_tensor(c, dtype, rank, k, kind, seed) for k, c in enumerate(counts)]


def all_ranks(counts, dtype, nranks, kind="normal", seed=SEED):
    """xs[r][k] for every simulated rank."""
    return [rank_tensors(counts, dtype, r, kind, seed) for r in range(nranks)]
