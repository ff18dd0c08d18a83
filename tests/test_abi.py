"""C-ABI library checks that need no GPU: it loads, exports every symbol declared
in include/dualip.h, its host planners equal the oracle's layout/shard plans bit
for bit, and compute entry points fail loudly without a GPU (no CPU fallback)."""
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    lib = os.path.join(ROOT, "paper_2603_04621_b200", "lib", "libdualip.so")
    if not os.path.exists(lib):
        from paper_2603_04621_b200.build import build
        build()
    from paper_2603_04621_b200 import _lib
    return _lib


def test_exports_every_declared_symbol(L):
    hdr = open(os.path.join(ROOT, "include", "dualip.h")).read()
    declared = set(re.findall(r"^\s*(?:const\s+)?[\w\s\*]*?\b(dl_\w+)\s*\(", hdr, flags=re.M))
    assert len(declared) >= 25
    syms = os.popen(f"nm -D --defined-only {L.LIB_PATH}").read()
    exported = set(re.findall(r" T (dl_\w+)", syms))
    assert declared <= exported, declared - exported
    assert declared == set(L.EXPORTED)
    assert L.dl_abi_version() == 3


def _lens_cases(rng):
    yield np.zeros(0, np.int64)
    yield np.array([0, 0, 0])
    yield np.array([1, 2, 3, 5, 8, 255, 256, 511, 512, 4095, 4096, 70000])
    for _ in range(40):
        n = int(rng.integers(1, 3000))
        kind = rng.integers(0, 3)
        if kind == 0:
            lens = rng.poisson(rng.choice([2, 30, 100, 200]), n)
        elif kind == 1:
            lens = np.minimum((rng.pareto(1.0, n) + 1).astype(np.int64), 20000)
        else:
            lens = rng.integers(0, 600, n)
        lens[rng.random(n) < 0.03] = 0
        yield lens


def test_plan_tiles_equals_oracle(L):
    from oracle.layout import tile_plan
    rng = np.random.default_rng(0)
    for lens in _lens_cases(rng):
        rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
        for cap in (256, 492, 600, 2048):
            perm, off, tiles, total = L.dl_plan_tiles(rp, cap)
            operm, ooff, otiles, ototal = tile_plan(lens, cap)
            np.testing.assert_array_equal(perm, np.array(operm, np.int64))
            np.testing.assert_array_equal(off, np.array(ooff, np.int64))
            np.testing.assert_array_equal(tiles, np.array(otiles, np.int64).reshape(-1, 5))
            assert total == ototal


def test_plan_shards_equals_oracle(L):
    from oracle.layout import shard_bounds
    rng = np.random.default_rng(1)
    for lens in _lens_cases(rng):
        rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
        for W in (1, 2, 3, 4, 8):
            np.testing.assert_array_equal(L.dl_plan_shards(rp, W), np.array(shard_bounds(rp, W), np.int64))


def test_tile_cap_rule(L):
    for m in (1, 2, 3, 4):
        for J in (1, 50, 10_000, 24_000, 100_000):
            cap = L.dl_tile_cap(m, J)
            assert cap >= 256 and cap % 4 == 0 and cap <= 2048


def test_invalid_arguments_rejected(L):
    with pytest.raises(L.DualipError):
        L.dl_plan_tiles(np.array([0, 5, 3], np.int64), 512)          # decreasing row_ptr
    with pytest.raises(L.DualipError):
        L.dl_plan_tiles(np.array([0, 5], np.int64), 100)             # tile_cap below 256


def test_no_cpu_fallback(L):
    """Without a CUDA device, problem creation must fail with DL_ERR_CUDA."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present: covered by the gpu tests")
    rp = np.array([0, 1], np.int64)
    d = np.array([0], np.int32)
    f = np.ones(1, np.float32)
    desc = L.dl_problem_desc(1, 1, 1, 1, L.ptr(rp), L.ptr(d), L.ptr(f), L.ptr(f), L.ptr(f), None, 0, 1.0, 1.0, 0,
                             None)
    with pytest.raises(L.DualipError) as ei:
        L.dl_problem_create(desc)
    assert ei.value.status == 2
