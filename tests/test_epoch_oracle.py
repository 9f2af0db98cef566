"""The oracle's per-epoch functions (full-graph evaluation, cache refresh)
against fixtures made by the reference itself (tests/golden/make_golden_epoch.py).
CPU only."""

import numpy as np
import pytest

from conftest import epoch_graph, load_golden
from oracle import cache as ocache
from oracle import nn as onn
from oracle.philox import RefreshRng, refresh_uniforms

G = load_golden("epoch.npz")
EVAL = sorted({k.split("/")[1] for k in G if k.startswith("eval/")})
REFRESH = sorted({k.split("/")[2] for k in G if k.startswith("refresh/case/")})


@pytest.mark.parametrize("tag", EVAL)
@pytest.mark.parametrize("phase", [0, 1])
def test_oracle_full_forward_matches_reference(tag, phase):
    g = epoch_graph(G, str(G[f"eval/{tag}/graph"]))
    p = f"eval/{tag}/p{phase}"
    ws = [G[f"{p}/w{l}"] for l in range(3) if f"{p}/w{l}" in G]
    logits = onn.full_forward(g.row_offsets, g.col_indices, g.features, ws)
    assert np.array_equal(logits, G[f"{p}/logits"])
    for mask, key in ((g.val_mask, "val_acc"), (g.test_mask, "test_acc")):
        idx = np.flatnonzero(mask)
        acc = onn.accuracy(logits[idx], g.labels[idx]) if idx.size else 0.0
        assert acc == float(G[f"{p}/{key}"][0])


def test_oracle_cache_probs_match_reference():
    g = epoch_graph(G, "g2")
    assert np.array_equal(ocache.degree_probs(g.col_indices, g.num_nodes),
                          G["refresh/g2/degree_probs"])
    for fo, steps in ((5, 2), (10, 3)):
        ref = G[f"refresh/g2/walk_probs_f{fo}_s{steps}"]
        got = ocache.walk_probs(g.row_offsets, g.col_indices, g.train_mask, fo, steps)
        assert np.array_equal(got, ref)
    got = ocache.walk_probs(g.row_offsets, g.col_indices, G["refresh/g2small/train_mask"], 2, 1)
    assert np.array_equal(got, G["refresh/g2small/walk_probs_f2_s1"])
    assert (got == 0).any()  # unreachable nodes keep probability zero


@pytest.mark.parametrize("name", REFRESH)
def test_oracle_refresh_matches_reference(name):
    p = f"refresh/case/{name}"
    probs = G[str(G[f"{p}/probs_key"])]
    frac, seed, epoch = G[f"{p}/params"]
    ids = ocache.refresh_cache_ids(probs.size, probs, float(frac), RefreshRng(int(seed), int(epoch)))
    assert np.array_equal(ids, G[f"{p}/cached_ids"])
    assert ids.size == int(np.ceil(frac * probs.size))


def test_refresh_uniforms_contract():
    u = refresh_uniforms(3, 1, 1000)
    assert u.dtype == np.float64 and (u >= 0).all() and (u < 1).all()
    # 53-bit grid and stream independence from the sampling streams
    assert np.array_equal(u * 2.0 ** 53, np.floor(u * 2.0 ** 53))
    assert not np.array_equal(u[:10], refresh_uniforms(3, 2, 10))
    assert np.array_equal(u[:7], refresh_uniforms(3, 1, 7))


@pytest.mark.parametrize("name", ["g8", "rand", "hub"])
def test_oracle_build_csr_matches_reference(name):
    from oracle.sampler import build_csr, degree_bucket_features
    ro, col = build_csr(G[f"ingest/{name}/edges"], int(G[f"ingest/{name}/n"][0]))
    assert np.array_equal(ro, G[f"ingest/{name}/row_offsets"])
    assert np.array_equal(col, G[f"ingest/{name}/col_indices"])
    assert np.array_equal(degree_bucket_features(ro), G[f"ingest/{name}/features"])


def test_queue_sizing_formulas_match_reference():
    from paper_2601_04707_b200.autotune import (AutotuneError, compute_cap, compute_queue_size,
                                                steady_slice)
    for total, peak, mb, cap in G["autotune/cap"]:
        if cap < 0:
            with pytest.raises(AutotuneError):
                compute_cap(total, peak, mb)
        else:
            assert compute_cap(total, peak, mb) == int(cap)
    for prep, comp, cap, q in G["autotune/queue"]:
        assert compute_queue_size(prep, comp, int(cap)) == int(q)
    for n, a, b in G["autotune/steady"]:
        s = steady_slice(int(n))
        assert (s.start, s.stop) == (a, b)
