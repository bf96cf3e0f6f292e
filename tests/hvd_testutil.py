"""Shared test helpers: numpy (workloads format) <-> torch conversion, comparisons."""
import numpy as np

HVD_CODE = {"f32": 1, "bf16": 2, "i32": 3, "i64": 4}


def to_torch(x, dtype, device="cuda"):
    import torch
    if dtype == "bf16":
        t = torch.from_numpy(x.view(np.int16).copy()).view(torch.bfloat16)
    else:
        t = torch.from_numpy(x.copy())
    return t.to(device)


def from_torch(t, dtype):
    import torch
    t = t.detach().cpu()
    if dtype == "bf16":
        return t.view(torch.int16).numpy().view(np.uint16).copy()
    return t.numpy().copy()


def assert_same(got, ref, dtype, what=""):
    """Bitwise equality; NaN compared by class only (R10)."""
    assert got.shape == ref.shape, (what, got.shape, ref.shape)
    if dtype in ("i32", "i64"):
        bad = got != ref
    else:
        u = np.uint16 if dtype == "bf16" else np.uint32
        gb, rb = got.view(u), ref.view(u)
        if dtype == "bf16":
            gn = (gb & 0x7FFF) > 0x7F80
            rn = (rb & 0x7FFF) > 0x7F80
        else:
            gn = (gb & 0x7FFFFFFF) > 0x7F800000
            rn = (rb & 0x7FFFFFFF) > 0x7F800000
        bad = (gb != rb) & ~(gn & rn)
    if bad.any():
        i = int(np.flatnonzero(bad)[0])
        raise AssertionError(f"{what}: {int(bad.sum())} of {bad.size} elements differ; first at {i}: "
                             f"got {got[i]!r} want {ref[i]!r}")
