"""CPU-side checks of the C ABI: the library loads, exports every symbol the
header declares, and its host logic (fusion plan, chunk partition, argument
validation) agrees with the independently written oracle.  No GPU compute."""
import ctypes as C
import pathlib
import re
import subprocess

import numpy as np
import pytest

import oracle
import workloads

ROOT = pathlib.Path(__file__).resolve().parents[1]


@pytest.fixture(scope="module")
def L():
    from paper_1802_05799_b200 import _build
    _build.build()
    from paper_1802_05799_b200 import _lib
    return _lib


def _header_functions():
    text = (ROOT / "include" / "hvd.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(hvd_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol(L):
    declared = _header_functions()
    assert declared == L.EXPORTS
    out = subprocess.run(["nm", "-D", "--defined-only", str(L.LIB_PATH)], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r" T (hvd_\w+)", out))
    assert set(declared) <= exported


def test_library_build_id_matches_the_sources(L):
    """build() recompiles when any source changes: the library embeds the sha256 of its
    sources (hvd_build_id) and the loaded one is the tree's."""
    from paper_1802_05799_b200 import _build
    assert L.lib.hvd_build_id().decode() == "hvd-src-" + _build.source_hash()
    assert not _build._stale()


def test_build_hash_tracks_every_source(tmp_path, monkeypatch):
    """A change to any compiled file changes the build id (so a stale .so is rebuilt)."""
    import shutil
    from paper_1802_05799_b200 import _build
    h0 = _build.source_hash()
    src = tmp_path / "csrc"
    shutil.copytree(_build.CSRC, src)
    monkeypatch.setattr(_build, "CSRC", src)
    assert _build.source_hash() == h0
    for name in _build.SOURCES + _build.HEADERS:
        f = src / name
        old = f.read_bytes()
        f.write_bytes(old + b"\n// touched\n")
        assert _build.source_hash() != h0, name
        f.write_bytes(old)
    assert _build.source_hash() == h0


def test_library_is_sm100a(L):
    out = subprocess.run(["cuobjdump", "--list-elf", str(L.LIB_PATH)], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def _plan_via_abi(L, tensors, threshold, capacity):
    n = len(tensors)
    counts = (C.c_uint64 * max(1, n))(*[c for c, _ in tensors])
    codes = {"f32": 1, "bf16": 2, "i32": 3, "i64": 4}
    dts = (C.c_int32 * max(1, n))(*[codes[d] for _, d in tensors])
    ne, nb = C.c_int(0), C.c_int(0)
    st = L.lib.hvd_plan(counts, dts, n, threshold, capacity, None, C.byref(ne), None, C.byref(nb))
    assert st in (0, -1)
    ents = (L.hvd_plan_entry * max(1, ne.value))()
    bufs = (L.hvd_plan_buffer * max(1, nb.value))()
    L.check(L.lib.hvd_plan(counts, dts, n, threshold, capacity, ents, C.byref(ne), bufs, C.byref(nb)))
    inv = {v: k for k, v in codes.items()}
    out = []
    for b in bufs[:nb.value]:
        es = [(e.tensor, e.src_off, e.dst_off, e.count) for e in ents[b.first_entry:b.first_entry + b.n_entries]]
        out.append((inv[b.dtype], b.length, es))
    return out


def _plan_via_oracle(tensors, threshold, capacity):
    return [(b.dtype, b.length, [(e.tensor, e.src_off, e.dst_off, e.count) for e in b.entries])
            for b in oracle.fusion_plan(tensors, threshold, capacity)]


@pytest.mark.parametrize("model", ["resnet101", "inception_v3", "vgg16"])
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("threshold", [64 << 20, 0, 1 << 20])
def test_plan_parity_model_sets(L, model, dtype, threshold):
    tensors = [(c, dtype) for _, c in workloads.gradient_set(model)]
    assert _plan_via_abi(L, tensors, threshold, 64 << 20) == _plan_via_oracle(tensors, threshold, 64 << 20)


def test_plan_parity_random(L):
    rng = np.random.default_rng(11)
    dts = ["f32", "bf16", "i32", "i64"]
    for _ in range(400):
        n = int(rng.integers(0, 30))
        tensors = [(int(rng.integers(0, 500)), dts[int(rng.integers(0, 4))]) for _ in range(n)]
        cap = int(rng.choice([64, 256, 1024, 4096]))
        thr = int(rng.choice([0, 32, 100, 512, cap, 10 * cap]))
        assert _plan_via_abi(L, tensors, thr, cap) == _plan_via_oracle(tensors, thr, cap)


def test_chunk_bounds_parity(L):
    codes = {"f32": 1, "bf16": 2, "i32": 3, "i64": 4}
    for n in range(1, 9):
        for dt, code in codes.items():
            for length in [0, 1, 7, 63, 64, 65, 64 * n, 64 * n + 1, 12345, 16 << 20]:
                out = (C.c_uint64 * (n + 1))()
                L.check(L.lib.hvd_chunk_bounds(length, n, code, out))
                assert list(out) == oracle.chunk_bounds(length, n, dt)


def test_argument_errors_without_device(L):
    h = C.c_void_p()
    assert L.lib.hvd_init(0, 0, 0, 0, C.byref(h)) == L.HVD_ERR_INVALID
    assert L.lib.hvd_init(2, 2, 0, 0, C.byref(h)) == L.HVD_ERR_INVALID
    assert L.lib.hvd_init_virtual(9, 0, 0, C.byref(h)) == L.HVD_ERR_INVALID
    assert L.lib.hvd_allreduce(None, None, 0, 0, 0, None) == L.HVD_ERR_INVALID
    assert L.lib.hvd_poll_error(None) == L.HVD_ERR_INVALID
    assert L.lib.hvd_finalize(None) == 0
    out = (C.c_uint64 * 2)()
    assert L.lib.hvd_chunk_bounds(10, 1, 9, out) == L.HVD_ERR_UNSUPPORTED
    for s in (0, -1, -2, -3, -4, -5, -6):
        assert L.strerror(s)


def test_package_fails_loudly_without_library(tmp_path):
    """The product path has no fallback: a missing .so is an ImportError."""
    code = ("import sys, pathlib; sys.path.insert(0, %r);"
            "import paper_1802_05799_b200._lib as m" % str(tmp_path))
    pkg = tmp_path / "paper_1802_05799_b200"
    pkg.mkdir()
    (pkg / "__init__.py").write_text("")
    (pkg / "_lib.py").write_text((ROOT / "paper_1802_05799_b200" / "_lib.py").read_text())
    r = subprocess.run(["python", "-c", code], capture_output=True, text=True)
    assert r.returncode != 0 and "not built" in r.stderr


def test_product_does_not_import_oracle():
    for p in (ROOT / "paper_1802_05799_b200").rglob("*"):
        if p.suffix in (".py", ".cu", ".cpp", ".h"):
            txt = p.read_text()
            assert "import oracle" not in txt and "from oracle" not in txt and "oracle/" not in txt, p
