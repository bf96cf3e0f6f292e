"""Pins of the CPU oracle against what the paper and mathematics fix.

Every test here checks ``oracle/`` against something other than itself:
closed forms, invariants, library routines, brute force on tiny inputs,
golden values from SPEC.md / SURVEY.md (``tests/golden``).  A plausible
mistake in the oracle (dropped term, wrong sign or index, transposed
chunk, wrong rounding) fails at least one of them.

Pinned / unpinned summary (also DESIGN.md §Parity):
  * ring simulation: rotated-fold closed form, N=2 textbook, N=1 identity,
    brute force, traffic closed form, rank agreement       -> pinned
  * averaging: all-ones, rank-index, prescale == postscale  -> pinned
  * bf16 rounding: ml_dtypes / torch library casts          -> pinned
  * fusion plan: SPEC examples, invariants   -> pinned
  * chunk quantum, member alignment, oversize split         -> parity unpinned
"""
import json
import os

import ml_dtypes
import numpy as np
import pytest
import torch

import oracle
import workloads

GOLD = os.path.join(os.path.dirname(__file__), "golden")
DTYPES = ["f32", "bf16", "i32", "i64"]


def _load(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def _f64(x, dtype):
    """Exact widening to float64 (test-side, via library casts)."""
    with np.errstate(invalid="ignore"):
        if dtype == "bf16":
            return x.view(ml_dtypes.bfloat16).astype(np.float64)
        return x.astype(np.float64)


def _bits_equal_or_both_nan(a, b, dtype):
    if dtype in ("i32", "i64"):
        return np.array_equal(a, b)
    fa, fb = _f64(a, dtype), _f64(b, dtype)
    both_nan = np.isnan(fa) & np.isnan(fb)
    same = a.view(np.uint16 if dtype == "bf16" else np.uint32) == b.view(np.uint16 if dtype == "bf16" else np.uint32)
    return bool(np.all(same | both_nan))


# ---------------------------------------------------------------- bf16 casts
def test_bf16_rne_matches_ml_dtypes():
    rng = np.random.default_rng(1)
    u = rng.integers(0, 2**32, size=1 << 20, dtype=np.uint64).astype(np.uint32)
    edge = np.array([0, 0x80000000, 0x7F7FFFFF, 0xFF7FFFFF, 0x7F800000, 0xFF800000,
                     0x00000001, 0x807FFFFF, 0x3F808000, 0x3F818000, 0x3F80FFFF,
                     0x3F817FFF, 0x7F7F8000, 0x7FC00000, 0x7F800001], dtype=np.uint32)
    x = np.concatenate([u, edge]).view(np.float32)
    got = oracle.f32_to_bf16_rne(x)
    with np.errstate(invalid="ignore"):
        ref = x.astype(ml_dtypes.bfloat16).view(np.uint16)
    assert _bits_equal_or_both_nan(got, ref, "bf16")


def test_bf16_widen_is_exact():
    h = np.arange(0, 1 << 16, dtype=np.uint32).astype(np.uint16)
    got = oracle.bf16_to_f32(h)
    ref = h.view(ml_dtypes.bfloat16).astype(np.float32)
    assert _bits_equal_or_both_nan(got, ref, "f32")


def test_bf16_add_matches_torch_cpu():
    rng = np.random.default_rng(2)
    a = rng.standard_normal(1 << 18).astype(np.float32) * np.float32(8)
    b = rng.standard_normal(1 << 18).astype(np.float32)
    ah = a.astype(ml_dtypes.bfloat16).view(np.uint16)
    bh = b.astype(ml_dtypes.bfloat16).view(np.uint16)
    got = oracle.add_w(ah, bh, "bf16")
    ta = torch.from_numpy(ah.view(np.int16)).view(torch.bfloat16)
    tb = torch.from_numpy(bh.view(np.int16)).view(torch.bfloat16)
    ref = (ta + tb).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(got, ref)


# ---------------------------------------------------------------- fusion plan
def test_fusion_plan_spec_examples():
    g = _load("spec_fusion_examples.json")
    c0, c1, c2 = g["cases"]
    p = oracle.fusion_plan([tuple(t) for t in c0["tensors"]], c0["threshold"])
    assert [[e.tensor for e in b.entries] for b in p] == c0["expect_groups"]
    p = oracle.fusion_plan([(256, "f32")] * 1000, c1["threshold"])
    assert len(p) == 1 and len(p[0].entries) == 1000
    assert p[0].length * 4 == c1["expect_bytes"]
    p = oracle.fusion_plan([tuple(t) for t in c2["tensors"]], c2["threshold"])
    assert [[e.tensor for e in b.entries] for b in p] == c2["expect_groups"]


@pytest.mark.parametrize("model", ["resnet101", "inception_v3", "vgg16"])
def test_fusion_plan_survey_model_sets(model):
    g = _load("survey_model_plans.json")
    ref = g["models"][model]
    gs = workloads.gradient_set(model)
    assert len(gs) == ref["tensors"]
    assert sum(c for _, c in gs) == ref["params"]
    for dt, key in (("f32", "f32_mib"), ("bf16", "bf16_mib")):
        p = oracle.fusion_plan([(c, dt) for _, c in gs])
        mib = [b.length * oracle.ELEM_SIZE[dt] / 2**20 for b in p]
        assert len(mib) == len(ref[key])
        assert np.allclose(mib, ref[key], atol=g["tolerance_mib"])


def _check_plan_invariants(tensors, threshold, capacity, plan):
    limit = capacity if threshold == 0 else min(threshold, capacity)
    covered = [0] * len(tensors)
    order = []
    for b in plan:
        esz = oracle.ELEM_SIZE[b.dtype]
        assert b.length * esz <= limit
        if threshold == 0:
            assert len(b.entries) == 1
        end = 0
        for e in b.entries:
            assert tensors[e.tensor][1] == b.dtype            # same data type
            assert (e.dst_off * esz) % 16 == 0
            assert e.dst_off >= end
            end = e.dst_off + e.count
            assert e.src_off == covered[e.tensor]             # contiguous, in order
            covered[e.tensor] += e.count
            order.append(e.tensor)
        assert end == b.length
    assert covered == [c for c, _ in tensors]
    assert order == sorted(order)                             # submission order kept
    # next-fit maximality: the first member of buffer i+1 did not fit buffer i
    for a, b in zip(plan, plan[1:]):
        if threshold == 0 or a.dtype != b.dtype:
            continue
        e = b.entries[0]
        esz = oracle.ELEM_SIZE[b.dtype]
        last = a.entries[-1]
        if e.src_off != 0 or last.src_off != 0 or last.count != tensors[last.tensor][0]:
            continue  # split segments of an oversize tensor are singleton buffers (R7)
        off = -(-a.length * esz // 16) * 16
        assert off + tensors[e.tensor][0] * esz > limit


def test_fusion_plan_invariants_random():
    rng = np.random.default_rng(3)
    for trial in range(300):
        n = int(rng.integers(0, 40))
        tensors = [(int(rng.integers(0, 300)), DTYPES[int(rng.integers(0, 2 if trial % 2 else 4))])
                   for _ in range(n)]
        cap = int(rng.choice([64, 128, 1000, 4096]))
        thr = int(rng.choice([0, 16, 100, 512, cap]))
        plan = oracle.fusion_plan(tensors, thr, cap)
        _check_plan_invariants(tensors, thr, cap, plan)


def test_fusion_off_is_one_buffer_per_tensor():
    tensors = [(5, "f32"), (0, "f32"), (7, "f32"), (3, "bf16")]
    p = oracle.fusion_plan(tensors, 0)
    assert [[e.tensor for e in b.entries] for b in p] == [[0], [2], [3]]


def test_fits_is_inclusive_and_oversize_split():
    # VGG-16 fc7 is exactly 64 MiB: it must be one buffer (R6)
    p = oracle.fusion_plan([(4096 * 4096, "f32")])
    assert len(p) == 1 and p[0].length == 4096 * 4096
    # fc6 (392 MiB) -> 6 x 64 MiB + 8 MiB (R7)
    p = oracle.fusion_plan([(4096 * 25088, "f32")])
    assert [b.length * 4 // 2**20 for b in p] == [64] * 6 + [8]


# ---------------------------------------------------------------- chunk partition
def test_chunk_bounds_invariants():
    for n in range(1, 9):
        for dt in DTYPES:
            g = 256 // oracle.ELEM_SIZE[dt]
            for L in list(range(0, 3 * n * g + 5)) + [10**6 + 3]:
                b = oracle.chunk_bounds(L, n, dt)
                assert len(b) == n + 1 and b[0] == 0 and b[-1] == L
                assert all(x <= y for x, y in zip(b, b[1:]))
                assert all(x % g == 0 or x == L for x in b[:-1])
                sizes = [y - x for x, y in zip(b, b[1:])]
                q = max(sizes)
                full = [z for z in sizes if z]
                assert all(z == q for z in full[:-1])           # equal chunks, ragged last
                if L:
                    assert n * q >= L and (q <= g or n * (q - g) < L)  # smallest quantum multiple


# ---------------------------------------------------------------- ring simulation
def _ring(xs, dtype, op="sum"):
    outs, traffic = oracle.allreduce_buffer([x.copy() for x in xs], dtype, op)
    return outs, traffic


def _rotated_fold(xs, dtype, op):
    """Closed form: chunk c is the left fold x_c, x_{c+1}, ..., x_{c+N-1}.

    Written here without message passing: index arithmetic only.
    """
    n = len(xs)
    L = len(xs[0])
    if op == "average":
        s = np.float32(1.0) / np.float32(n)
        if dtype == "f32":
            xs = [(x * s).astype(np.float32) for x in xs]
        else:
            xs = [(x.view(ml_dtypes.bfloat16).astype(np.float32) * s).astype(ml_dtypes.bfloat16).view(np.uint16)
                  for x in xs]
    b = oracle.chunk_bounds(L, n, dtype)
    y = np.empty_like(xs[0])
    for c in range(n):
        sl = slice(b[c], b[c + 1])
        acc = xs[c][sl].copy()
        for j in range(1, n):
            v = xs[(c + j) % n][sl]
            if dtype == "f32":
                acc = (acc + v).astype(np.float32)
            elif dtype == "bf16":
                t = acc.view(ml_dtypes.bfloat16).astype(np.float32) + v.view(ml_dtypes.bfloat16).astype(np.float32)
                acc = t.astype(ml_dtypes.bfloat16).view(np.uint16)
            else:
                acc = (acc + v).astype(acc.dtype)
        y[sl] = acc
    return y


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 8])
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("op", ["sum", "average"])
def test_ring_equals_rotated_fold(n, dtype, op):
    for L in (0, 1, 63, 64 * n + 7, 100_003):
        xs = [workloads.rank_tensor(L, dtype, r, 0) for r in range(n)]
        outs, _ = _ring(xs, dtype, op)
        ref = _rotated_fold(xs, dtype, op)
        for r in range(n):
            assert _bits_equal_or_both_nan(outs[r], ref, dtype), (n, L, r)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_n2_textbook_average(dtype):
    """N=2: y = fl(x0/2 + x1/2) = fl(x0 + x1)/2 exactly, whatever the chunks."""
    xs = [workloads.rank_tensor(50_001, dtype, r, 3) for r in range(2)]
    outs, _ = _ring(xs, dtype, "average")
    if dtype == "f32":
        ref = ((xs[0] + xs[1]).astype(np.float32) * np.float32(0.5)).astype(np.float32)
    else:
        a = xs[0].view(ml_dtypes.bfloat16).astype(np.float32)
        b = xs[1].view(ml_dtypes.bfloat16).astype(np.float32)
        ref = ((a + b).astype(ml_dtypes.bfloat16).astype(np.float32) * np.float32(0.5)).astype(
            ml_dtypes.bfloat16).view(np.uint16)
    assert _bits_equal_or_both_nan(outs[0], ref, dtype)
    assert _bits_equal_or_both_nan(outs[1], ref, dtype)


@pytest.mark.parametrize("dtype", DTYPES)
def test_n1_identity(dtype):
    kind = "normal" if dtype in ("f32", "bf16") else "int_uniform"
    x = workloads.rank_tensor(1000, dtype, 0, 0, kind)
    outs, tr = _ring([x], dtype, "sum")
    assert np.array_equal(outs[0].view(np.uint8), x.view(np.uint8)) and tr[0].sends == 0


@pytest.mark.parametrize("n", [2, 4, 8])
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_average_closed_forms(n, dtype):
    L = 64 * n * 3 + 5
    ones = [workloads.rank_tensor(L, dtype, r, 0, "ones") for r in range(n)]
    outs, _ = _ring(ones, dtype, "average")
    for o in outs:
        assert np.all(_f64(o, dtype) == 1.0)
    ri = [workloads.rank_tensor(L, dtype, r, 0, "rank_index") for r in range(n)]
    outs, _ = _ring(ri, dtype, "average")
    for o in outs:
        assert np.all(_f64(o, dtype) == (n - 1) / 2)


def test_rank_index_not_exact_for_n5_f32():
    """Sanity of the previous pin: with N=5, fl32(1/5) is inexact."""
    n, L = 5, 64 * 5 * 4
    ri = [workloads.rank_tensor(L, "f32", r, 0, "rank_index") for r in range(n)]
    outs, _ = _ring(ri, "f32", "average")
    assert not np.all(outs[0].astype(np.float64) == 2.0)


@pytest.mark.parametrize("n", [2, 4, 8])
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_prescale_equals_postscale_power_of_two(n, dtype):
    """R1: for power-of-two N, scaling by 1/N is exact, so average == sum * (1/N)."""
    xs = [workloads.rank_tensor(20_000, dtype, r, 5) for r in range(n)]
    avg, _ = _ring(xs, dtype, "average")
    sm, _ = _ring(xs, dtype, "sum")
    inv = 1.0 / n
    ref = _f64(sm[0], dtype) * inv
    assert np.array_equal(_f64(avg[0], dtype), ref)


@pytest.mark.parametrize("dtype", ["i32", "i64"])
@pytest.mark.parametrize("n", [1, 2, 3, 5, 8])
def test_integer_exact_and_permutation_invariant(dtype, n):
    L = 1000
    xs = [workloads.rank_tensor(L, dtype, r, 0, "int_uniform") for r in range(n)]
    if dtype == "i32":  # force wrap-around
        xs = [(x.astype(np.int64) * 4096).astype(np.int32) for x in xs]
    outs, _ = _ring(xs, dtype)
    total = np.sum(np.stack([x.astype(np.int64) for x in xs]), axis=0)
    if dtype == "i32":
        total = ((total + 2**31) % 2**32 - 2**31).astype(np.int32)
    for o in outs:
        assert np.array_equal(o, total.astype(o.dtype))
    perm = list(reversed(xs))
    outs2, _ = _ring(perm, dtype)
    assert np.array_equal(outs2[0], outs[0])


@pytest.mark.parametrize("n", [2, 3, 4, 8])
def test_fp_accuracy_vs_fp64(n):
    """|y - m| <= gamma * sum|x|/N elementwise (R5); fp32 within 1e-6."""
    L = 200_000
    for dtype, u in (("f32", 2.0**-24), ("bf16", 2.0**-8)):
        xs = [workloads.rank_tensor(L, dtype, r, 1) for r in range(n)]
        outs, _ = _ring(xs, dtype, "average")
        X = np.stack([_f64(x, dtype) for x in xs])
        m = X.sum(0) / n
        a = np.abs(X).sum(0) / n
        k = n  # N-1 adds + 1 prescale rounding
        gamma = k * u / (1 - k * u)
        err = np.abs(_f64(outs[0], dtype) - m)
        assert np.all(err <= gamma * a + 1e-300)
        if dtype == "f32":
            assert np.all(err <= 1e-6 * a + 1e-300)       # north_star fp32 bound
        else:
            nrm = np.linalg.norm(_f64(outs[0], dtype) - m) / np.linalg.norm(m)
            assert nrm <= 1e-2                           # north_star bf16, norm-wise (R5)


@pytest.mark.parametrize("n", range(1, 9))
def test_traffic_closed_form(n):
    for dtype in ("f32", "bf16"):
        for L in list(range(0, 3 * n + 3)) + [64 * n * 2 + 17, 10**6]:
            xs = [np.zeros(L, dtype=oracle.NP_TYPE[dtype]) for _ in range(n)]
            _, tr = _ring(xs, dtype)
            b = oracle.chunk_bounds(L, n, dtype)
            size = [b[c + 1] - b[c] for c in range(n)]
            for r in range(n):
                assert tr[r].sends == 2 * (n - 1)
                assert tr[r].sent_elems == (2 * L - size[(r + 1) % n] - size[(r + 2) % n] if n > 1 else 0)
                assert tr[r].recv_elems == (2 * L - size[r] - size[(r + 1) % n] if n > 1 else 0)
            assert sum(t.sent_elems for t in tr) == 2 * (n - 1) * L
            # bandwidth optimality bound
            g = 256 // oracle.ELEM_SIZE[dtype]
            for t in tr:
                assert t.sent_elems <= 2 * (n - 1) * (L / n) + 2 * (n - 1) * g


@pytest.mark.parametrize("n", range(1, 9))
def test_brute_force_tiny(n):
    for dtype in DTYPES:
        g = 256 // oracle.ELEM_SIZE[dtype]
        for L in list(range(0, 3 * n + 3)) + [g * n + 1]:
            xs = [workloads.rank_tensor(L, dtype, r, L, "small_int") for r in range(n)]
            outs, _ = _ring(xs, dtype)
            exact = np.zeros(L)
            for x in xs:
                exact += _f64(x, dtype)
            for o in outs:
                assert np.array_equal(_f64(o, dtype), exact)


def test_rank_agreement_specials():
    for n in (2, 3, 4, 8):
        for dtype in ("f32", "bf16"):
            xs = [workloads.rank_tensor(5000, dtype, r, 2, "specials") for r in range(n)]
            outs, _ = _ring(xs, dtype, "average")
            for o in outs[1:]:
                assert np.array_equal(o.view(np.uint8), outs[0].view(np.uint8))


# ---------------------------------------------------------------- whole path
def test_spec_golden_examples():
    g = _load("spec_ring_examples.json")
    for case in g["allreduce"]:
        dt = case["dtype"]
        xs = [[np.array(v, dtype=oracle.NP_TYPE[dt])] for v in case["inputs"]]
        outs, tr, _ = oracle.allreduce(xs, [dt], case["op"])
        for r in range(case["N"]):
            assert outs[r][0].tolist() == case["expect"]
            assert tr[r].sends == case["sends_per_rank"]
    for case in g["broadcast"]:
        n, root = case["N"], case["root"]
        xs = [[np.array(case["root_input"] if r == root else [0, 0, 0], dtype=np.int32)] for r in range(n)]
        outs, _ = oracle.broadcast(xs, root)
        assert all(o[0].tolist() == case["expect"] for o in outs)


@pytest.mark.parametrize("n", [2, 3, 4])
def test_fused_equals_unfused_integers(n):
    counts = [5, 64, 1, 300, 17, 0, 129]
    for dtype in ("i32", "i64"):
        xs = [workloads.rank_tensors(counts, dtype, r, "int_uniform") for r in range(n)]
        fused, _, p1 = oracle.allreduce(xs, [dtype] * len(counts), "sum", threshold=1 << 20)
        unfused, _, p2 = oracle.allreduce(xs, [dtype] * len(counts), "sum", threshold=0)
        assert len(p1) == 1 and len(p2) == 6
        for r in range(n):
            for a, b in zip(fused[r], unfused[r]):
                assert np.array_equal(a, b)


@pytest.mark.parametrize("n", [2, 4])
def test_fused_f32_within_bound_of_unfused(n):
    counts = [33, 1000, 4, 2048]
    xs = [workloads.rank_tensors(counts, "f32", r) for r in range(n)]
    f, _, _ = oracle.allreduce(xs, ["f32"] * 4, "average", threshold=1 << 20)
    u, _, _ = oracle.allreduce(xs, ["f32"] * 4, "average", threshold=0)
    for a, b, k in zip(f[0], u[0], range(4)):
        scale = np.abs(np.stack([xs[r][k] for r in range(n)])).astype(np.float64).sum(0) / n
        assert np.all(np.abs(a.astype(np.float64) - b) <= 1e-6 * scale + 1e-300)


def test_pack_unpack_roundtrip_is_lossless():
    """Copy-in / copy-out is bitwise lossless at N=1."""
    counts = [3, 8, 0, 1025, 64]
    for dtype in DTYPES:
        kind = "normal" if dtype in ("f32", "bf16") else "int_uniform"
        xs = [workloads.rank_tensors(counts, dtype, 0, kind)]
        outs, _, _ = oracle.allreduce(xs, [dtype] * len(counts), "sum", threshold=512)
        for a, b in zip(outs[0], xs[0]):
            assert np.array_equal(a.view(np.uint8), b.view(np.uint8))


def test_mixed_dtype_list_end_to_end():
    counts = [10, 20, 30, 40]
    dts = ["f32", "bf16", "f32", "bf16"]
    n = 3
    xs = [[workloads.rank_tensor(c, d, r, k, "small_int") for k, (c, d) in enumerate(zip(counts, dts))]
          for r in range(n)]
    outs, _, plan = oracle.allreduce(xs, dts, "sum")
    assert len(plan) == 4
    for k in range(4):
        exact = sum(_f64(xs[r][k], dts[k]) for r in range(n))
        assert np.array_equal(_f64(outs[1][k], dts[k]), exact)


def test_average_rejects_integers():
    with pytest.raises(ValueError):
        oracle.allreduce([[np.zeros(4, np.int32)]] * 2, ["i32"], "average")


# ---------------------------------------------------------------- broadcast / allgather
@pytest.mark.parametrize("n", [1, 2, 3, 5, 8])
def test_broadcast_bitwise_and_idempotent(n):
    for root in range(n):
        xs = [workloads.rank_tensors([7, 300], "f32", r, "specials") for r in range(n)]
        outs, tr = oracle.broadcast(xs, root)
        for o in outs:
            for a, b in zip(o, xs[root]):
                assert np.array_equal(a.view(np.uint8), b.view(np.uint8))
        again, _ = oracle.broadcast(outs, root)
        for a, b in zip(again, outs):
            assert all(np.array_equal(p.view(np.uint8), q.view(np.uint8)) for p, q in zip(a, b))
        for r in range(n):
            assert tr[r].recv_elems == (0 if r == root else 307)
            assert tr[r].sent_elems == (0 if (r + 1) % n == root else 307)


@pytest.mark.parametrize("n", [1, 2, 3, 4, 8])
def test_allgather_is_rank_order_concatenation(n):
    xs = [workloads.rank_tensor(37, "i64", r, 0, "int_uniform") for r in range(n)]
    outs, tr = oracle.allgather(xs)
    ref = np.concatenate(xs)
    for o in outs:
        assert np.array_equal(o, ref)
    for t in tr:
        assert t.sent_elems == (n - 1) * 37 and t.recv_elems == (n - 1) * 37


# ---------------------------------------------------------------- wire-dtype variants
def test_bf16_wire_for_f32_n2_textbook():
    """N=2, fp32 grads, bf16 wire: y = f32( rne( f32(rne(x0/2)) + f32(rne(x1/2)) ) ), chunk-independent."""
    xs = [[workloads.rank_tensor(30_001, "f32", r, 0)] for r in range(2)]
    outs, _, _ = oracle.allreduce(xs, ["f32"], "average", wire="bf16")
    h = [(x[0] * np.float32(0.5)).astype(ml_dtypes.bfloat16).astype(np.float32) for x in xs]
    ref = (h[0] + h[1]).astype(ml_dtypes.bfloat16).astype(np.float32)
    for r in range(2):
        assert np.array_equal(outs[r][0].view(np.uint32), ref.view(np.uint32))


def test_f32_wire_for_bf16_rotated_fold():
    """bf16 grads, fp32 wire: chunk c = rne( fold_fp32(f32(x_j) * s) ), one final rounding."""
    n, L = 4, 70_001
    xs = [[workloads.rank_tensor(L, "bf16", r, 2)] for r in range(n)]
    outs, _, plan = oracle.allreduce(xs, ["bf16"], "average", wire="f32")
    s = np.float32(1.0) / np.float32(n)
    w = [(x[0].view(ml_dtypes.bfloat16).astype(np.float32) * s).astype(np.float32) for x in xs]
    b = oracle.chunk_bounds(L, n, "f32")
    ref = np.empty(L, dtype=np.float32)
    for c in range(n):
        sl = slice(b[c], b[c + 1])
        acc = w[c][sl].copy()
        for j in range(1, n):
            acc = (acc + w[(c + j) % n][sl]).astype(np.float32)
        ref[sl] = acc
    ref16 = ref.astype(ml_dtypes.bfloat16).view(np.uint16)
    for r in range(n):
        assert np.array_equal(outs[r][0], ref16)


@pytest.mark.parametrize("n", [2, 4, 8])
def test_wire_variant_accuracy(n):
    """bf16 grads with fp32 partials meet north_star's 1e-2 elementwise (R5 note); bf16 wire for
    fp32 grads stays within the bf16 gamma bound."""
    L = 100_000
    xs = [[workloads.rank_tensor(L, "bf16", r, 1)] for r in range(n)]
    outs, _, _ = oracle.allreduce(xs, ["bf16"], "average", wire="f32")
    X = np.stack([_f64(x[0], "bf16") for x in xs])
    m, a = X.sum(0) / n, np.abs(X).sum(0) / n
    assert np.all(np.abs(_f64(outs[0][0], "bf16") - m) <= 1e-2 * a + 1e-300)
    xf = [[workloads.rank_tensor(L, "f32", r, 1)] for r in range(n)]
    outs, _, _ = oracle.allreduce(xf, ["f32"], "average", wire="bf16")
    X = np.stack([x[0].astype(np.float64) for x in xf])
    m, a = X.sum(0) / n, np.abs(X).sum(0) / n
    k = n + 1
    u = 2.0 ** -8
    assert np.all(np.abs(outs[0][0].astype(np.float64) - m) <= k * u / (1 - k * u) * a + 1e-300)


def test_wire_plan_uses_wire_bytes():
    """64 MiB of bf16 wire holds 32 Mi fp32 gradient elements: fusion limits count wire bytes."""
    p = oracle.fusion_plan([(24 << 20, "bf16")])
    assert len(p) == 1
    p32 = oracle.fusion_plan([(24 << 20, "f32")])
    assert len(p32) == 2
