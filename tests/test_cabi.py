"""The C-ABI library: exports, host-side entry points, error reporting (no GPU)."""

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

from oracle.philox import draws, fisher_yates_positions

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "mqgnn.h"


def header_symbols():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(mq_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def L():
    from paper_2601_04707_b200 import _build
    from paper_2601_04707_b200._lib import lib
    _build.build()  # incremental: no-op when up to date
    return lib()


def test_every_header_symbol_is_exported_and_bound(L):
    from paper_2601_04707_b200._lib import SIGNATURES
    syms = header_symbols()
    assert len(syms) >= 30
    for s in syms:
        assert hasattr(L.dll, s), f"{s} not exported by libmqgnn.so"
        assert s in SIGNATURES, f"{s} has no ctypes signature"
    assert set(SIGNATURES) == set(syms)


def test_version_and_scratch_queries(L):
    assert L.mq_version() == 1
    assert L.mq_scan_scratch_bytes(1) > 0
    assert L.mq_scan_scratch_bytes(10**8) > L.mq_scan_scratch_bytes(10**4)
    assert L.mq_relabel_scratch_bytes(1024, 10) > 0
    assert L.mq_linear_scratch_bytes(2722, 602, 64) >= 2 * 602 * 64 * 4
    assert L.mq_prof_num_kernels() > 20
    names = {L.mq_prof_kernel_name(i).decode() for i in range(L.mq_prof_num_kernels())}
    assert {"sample_hop", "gather", "spmm_fwd", "linear_fwd", "adam"} <= names


@pytest.mark.parametrize("key", [(0, 0, 0, 0, 0), (7, 3, 11, 1, 5), (2**40 + 5, 9, 123, 2, 999)])
def test_host_philox_matches_oracle(L, key):
    out = np.zeros(37, dtype=np.uint32)
    L.mq_philox_fill_host(*key, 37, out.ctypes.data)
    assert np.array_equal(out, draws(*key, count=37))


@pytest.mark.parametrize("n,k", [(10, 10), (100, 3), (2**31 - 5, 15), (33, 32), (1, 1)])
def test_host_fisher_yates_matches_oracle(L, n, k):
    pos = np.zeros(k, dtype=np.int64)
    L.mq_fisher_yates_host(3, 4, 5, 6, 7, n, k, pos.ctypes.data)
    assert pos.tolist() == fisher_yates_positions(draws(3, 4, 5, 6, 7, k), n, k)


def test_errors_are_reported(L):
    from paper_2601_04707_b200._lib import MQError
    pos = np.zeros(4, dtype=np.int64)
    with pytest.raises(MQError, match="k=4 > n=3"):
        L.mq_fisher_yates_host(0, 0, 0, 0, 0, 3, 4, pos.ctypes.data)
    with pytest.raises(MQError, match="fanout"):
        L.mq_sample_hop(None, None, None, None, None, None, 1, 0, 0, 0, 0, 0, None, None, None,
                        None)
    assert b"fanout" in L.dll.mq_last_error()


def test_missing_library_fails_loudly(tmp_path, monkeypatch):
    from paper_2601_04707_b200 import _lib
    with pytest.raises(_lib.MQError, match="no CPU fallback"):
        _lib._Lib(tmp_path / "nope.so")


@pytest.mark.parametrize("seed,epoch,n", [(3, 1, 1000), (2**40 + 7, 9, 77), (0, 0, 1)])
def test_host_refresh_uniforms_match_oracle(L, seed, epoch, n):
    from oracle.philox import refresh_uniforms
    out = np.zeros(n, dtype=np.float64)
    L.mq_refresh_uniforms_host(seed, epoch, n, out.ctypes.data)
    assert np.array_equal(out, refresh_uniforms(seed, epoch, n))


def test_eval_and_refresh_scratch_queries(L):
    assert L.mq_full_agg_scratch_bytes(10**8, 64) >= 2 * (10**8 // 1024) * 64 * 4
    # one split (>= 148 row tiles): the GEMM writes y directly, no partials
    assert L.mq_full_transform_part_floats(232965, 64) == 1
    assert L.mq_full_transform_part_floats(5000, 64) >= 5000 * 128
    assert L.mq_walk_scratch_bytes(10**6) >= 3 * 8 * 10**6
    assert L.mq_refresh_scratch_bytes(10**6) >= 12 * 10**6


def test_gemm_kernel_selection_is_validated(L):
    """mq_set_tc_kernel: 1 (cp.async), 2 (TMA, default), 3 (TMA for every
    mode); anything else is an argument error and leaves the choice alone."""
    from paper_2601_04707_b200._lib import MQError
    old = L.mq_get_tc_kernel()
    assert old == 2
    try:
        for v in (1, 3, 2):
            L.mq_set_tc_kernel(v)
            assert L.mq_get_tc_kernel() == v
        with pytest.raises(MQError, match="mq_set_tc_kernel"):
            L.mq_set_tc_kernel(4)
        assert L.mq_get_tc_kernel() == 2
    finally:
        L.mq_set_tc_kernel(old)
