"""CPU-only checks of the native pieces (no GPU needed).

* the C-ABI library loads and exports every symbol include/bittrain_b200.h declares;
* the device arithmetic headers, compiled for the host, are bit-exact with the
  host libm (tanh) and with the oracle (fold shapes);
* the native host helpers (Fisher-Yates, FNV, epoch deal, arrival order,
  rotation table) match the reference's golden vectors.
"""

import ctypes as C
import math
import re
import subprocess
from pathlib import Path

import numpy as np
import pytest

from golden_util import load, u64

ROOT = Path(__file__).resolve().parent.parent


def test_header_symbols_exported():
    from paper_2208_14228_b200 import _native

    header = (ROOT / "include" / "bittrain_b200.h").read_text()
    declared = set(re.findall(r"\b(bt_\w+)\s*\(", header))
    assert len(declared) >= 30
    lib = _native.lib()  # loads without a GPU
    missing = [s for s in sorted(declared) if not hasattr(lib, s)]
    assert not missing, missing
    assert set(_native.EXPORTS) == declared
    out = subprocess.run(["nm", "-D", "--defined-only", str(_native.LIB_PATH)], capture_output=True, text=True).stdout
    for s in declared:
        assert re.search(rf"\bT {s}$", out, re.M), s
    assert lib.bt_abi_version() == 1


def test_library_targets_sm100a():
    from paper_2208_14228_b200 import _native

    out = subprocess.run(["cuobjdump", "--list-elf", str(_native.LIB_PATH)], capture_output=True, text=True).stdout
    assert "sm_100a" in out


@pytest.fixture(scope="module")
def shim(tmp_path_factory):
    so = tmp_path_factory.mktemp("shim") / "shim.so"
    subprocess.run(["g++", "-O2", "-std=c++17", "-fPIC", "-shared", "-ffp-contract=off", "-o", str(so),
                    str(ROOT / "tests" / "native" / "host_shim.cpp")], check=True)
    L = C.CDLL(str(so))
    for f in ("shim_tanh", "shim_tanh_simt", "shim_expm1"):
        getattr(L, f).restype = C.c_double
        getattr(L, f).argtypes = [C.c_double]
    L.shim_streamfold.restype = C.c_double
    L.shim_streamfold.argtypes = [C.POINTER(C.c_double), C.c_int, C.c_int]
    L.shim_streamfold_f32.restype = C.c_float
    L.shim_streamfold_f32.argtypes = [C.POINTER(C.c_float), C.c_int, C.c_int]
    return L


def test_libm_restatement_bitexact_on_host(shim):
    """bt_libm.cuh compiled for the host == this host's libm tanh/expm1 (the reference's math.tanh)."""
    rng = np.random.default_rng(2208)
    xs = np.concatenate([rng.uniform(-4, 4, 150_000), rng.uniform(-40, 40, 50_000), rng.uniform(-1e-4, 1e-4, 20_000),
                         rng.integers(0, 2**63, 30_000, dtype=np.int64).view(np.float64),
                         np.array([0.0, -0.0, np.inf, -np.inf, 22.0, 1e-300, 0.34657359027997264])])
    xs = xs[np.isfinite(xs) | np.isinf(xs)]
    want = np.array([math.tanh(float(x)) for x in xs])  # math.tanh == libm (np.tanh is numpy SIMD, not libm)
    for fn in (shim.shim_tanh, shim.shim_tanh_simt):  # scalar glibc form and the branch-free SIMT form
        got = np.array([fn(float(x)) for x in xs])
        assert np.array_equal(got.view(np.uint64), want.view(np.uint64))
    ys = xs[np.abs(xs) < 400] * 1.7
    got = np.array([shim.shim_expm1(float(y)) for y in ys])
    assert np.array_equal(got.view(np.uint64), np.array([math.expm1(float(y)) for y in ys]).view(np.uint64))


def test_streamfold_equals_reference_tree(shim, oracle):
    rng = np.random.default_rng(5)
    for n in list(range(0, 40)) + [63, 64, 65, 100, 127, 128, 129, 255, 256, 1000]:
        v = rng.uniform(-1, 1, n) * 10.0 ** rng.integers(-12, 13, n)
        arr = (C.c_double * max(n, 1))(*v)
        for fan in (0, 2, 3, 4, 5, 7, 16, 64):
            want = oracle.reduce_sum(v, "seq" if fan == 0 else f"tree{fan}")
            got = shim.shim_streamfold(arr, n, fan)
            assert np.float64(got).view(np.uint64) == np.float64(want).view(np.uint64), (n, fan)


def test_compile_time_tree_equals_reference_tree(shim, oracle):
    rng = np.random.default_rng(6)
    for n in (1, 2, 4, 8, 16, 32, 64, 5, 12):
        v = rng.uniform(-1, 1, n) * 10.0 ** rng.integers(-12, 13, n)
        arr = (C.c_double * n)(*v)
        for kind, tag in (("tree2", "tree2"), ("seq", "seq")):
            fn = getattr(shim, f"shim_{kind}_{n}")
            fn.restype = C.c_double
            fn.argtypes = [C.POINTER(C.c_double)]
            assert np.float64(fn(arr)).view(np.uint64) == np.float64(oracle.reduce_sum(v, tag)).view(np.uint64)


def test_native_host_helpers_golden():
    import paper_2208_14228_b200 as bt
    from paper_2208_14228_b200.sampling import SamplePlan

    doc = load("prng.json")
    for c in doc["shuffled_range"]:
        assert bt.shuffled_range(c["n"], u64(c["state"])) == c["perm"]
    for c in doc["fnv1a64"]:
        assert bt.fnv1a64(bytes.fromhex(c["hex"])) == u64(c["hash"])
    for c in doc["derive_stream"]:
        assert bt.derive_stream(*[int(w, 16) for w in c["words"]]) == u64(c["state"])
    for c in doc["layout_arrival_perm"]:
        assert bt.layout_arrival_perm(c["n"], [tuple(x) for x in c["layout"]]) == c["perm"]
    for c in load("sampling.json")["epoch_indices"]:
        plan = SamplePlan(c["seed"], c["epoch"], c["n"], c["workers"], c["micro"], c["shuffle"])
        assert bt.epoch_indices(plan) == c["lists"]
    state, out = bt.splitmix64_next(0)
    assert out == 0xE220A8397B1DCDAF


def test_fused_launch_planning():
    """Which jobs take the one-launch fused step vs the per-seam kernels (host-only query)."""
    from types import SimpleNamespace

    from paper_2208_14228_b200.engine import _fused_fits

    def fits(E, B):
        return _fused_fits(SimpleNamespace(max_workers=E, micro_batch=B))

    assert fits(8, 4) and fits(64, 4) and fits(96, 2) and fits(2, 33)
    assert not fits(300, 4) and not fits(257, 1)


def test_rotation_table_matches_oracle(oracle):
    import paper_2208_14228_b200 as bt
    from paper_2208_14228_b200.buckets import rotation_table

    for c in load("allreduce.json")["cases"]:
        bm = bt.BucketMap(c["capacity"], tuple(tuple(b) for b in c["buckets"]))
        nrep = len(c["replicas"])
        assert rotation_table(bm, nrep).tolist() == oracle.rotation_table(c["buckets"], nrep, bm.param_count).tolist()


def test_model_stack_entry_points_validate_before_the_device():
    """The C3/C4 entry points reject malformed shapes with InputError (status 1) before any device call,
    so the checks run here without a GPU (the pointers are never dereferenced)."""
    from paper_2208_14228_b200 import _native
    from paper_2208_14228_b200.errors import InputError

    L = _native.lib()
    P, Q = 0x10000, 0x20000  # 16-byte aligned, never touched
    cases = [
        ("bt_gemm_conv", L.bt_gemm_conv(0, P, 1, 8, 8, 24, 8, 8, 3, 3, 1, 1, Q, P, 64, 1, 0, 0, 1, None)),  # Ci % 64
        ("bt_gemm_conv", L.bt_gemm_conv(1, P, 2, 8, 8, 64, 8, 8, 3, 3, 1, 1, Q, P, 64, 2, 100, 64 * 576, 0, None)),
        ("bt_cnn_upsample", L.bt_cnn_upsample(P, 1, 4, 4, 24, 2, Q, None)),  # C not a power of two
        ("bt_cnn_upsample", L.bt_cnn_upsample(P, 1, 4, 4, 64, 3, Q, None)),  # stride 3
        ("bt_cnn_bn_stats", L.bt_cnn_bn_stats(0, P, None, None, Q, Q, None, None, P, None, None, 0, None, None, 0,
                                              1, 64, 96, 1e-5, None)),  # C = 96
        ("bt_cnn_bn_apply", L.bt_cnn_bn_apply(P, None, Q, Q, Q + 4, Q, 1, 64, 64, 1, P, None)),  # misaligned gamma
        ("bt_fold_splits", L.bt_fold_splits(P, 1, 2, 6, Q, 6, None)),  # n % 4
    ]
    for name, status in cases:
        assert status == 1, (name, status)
        with pytest.raises(InputError):
            _native.check(status, name)


def test_native_fisher_yates_equals_oracle_across_sizes():
    """bt_host_shuffled_range equals the oracle's Fisher-Yates (prng.py:81-93) for tiny, typical, odd and
    large sizes and extreme states (the golden vectors pin a few small cases only)."""
    import sys

    import paper_2208_14228_b200 as bt

    sys.path.insert(0, str(ROOT / "oracle"))
    import oracle

    rng = np.random.default_rng(11)
    for n in (0, 1, 2, 3, 7, 64, 1000, 1024, 4097, 65_537, (1 << 20) + 5):
        for state in [0, 2**64 - 1] + [int(x) for x in rng.integers(0, 2**63, size=2, dtype=np.int64)]:
            a = bt.shuffled_range(n, state)
            b = oracle.shuffled_range(n, state) if n else []
            assert a == list(b), (n, state)
