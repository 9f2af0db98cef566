"""Pin the CPU oracle against vectors produced by the reference itself.

The golden fixtures were made by ``tests/golden/make_golden.py``, which runs
the unmodified reference (``mqpipe``) under the injected Philox draw contract.
These tests need no GPU.
"""

import json

import numpy as np
import pytest

from conftest import (GOLDEN, batch_prefixes, golden_batch, make_cfg1, make_g2, make_g8)
from oracle import cache as ocache
from oracle import nn as onn
from oracle import racom as oracom
from oracle import sampler as osamp
from oracle.philox import draws, fisher_yates_positions, philox4x32_10


def test_philox_known_answer_vectors():
    kat = json.loads((GOLDEN / "philox_kat.json").read_text())
    for v in kat["kat"]:
        got = philox4x32_10(np.array(v["ctr"]), np.array(v["key"])).tolist()
        assert got == v["out"]


def test_philox_streams_and_selection():
    kat = json.loads((GOLDEN / "philox_kat.json").read_text())
    for s in kat["streams"]:
        x = draws(s["seed"], s["epoch"], s["batch"], s["hop"], s["row"], s["k"])
        assert x.tolist() == s["draws"]
        pos = fisher_yates_positions(x, s["n"], s["k"])
        assert pos == s["positions"]
        assert len(set(pos)) == s["k"] and all(0 <= p < s["n"] for p in pos)


def _graph_for(prefix, golden):
    if prefix.startswith("g8"):
        return make_g8()
    if prefix.startswith("g2"):
        return make_g2(golden)
    return None


@pytest.fixture(scope="module")
def cfg1_graph():
    return make_cfg1()


def test_oracle_sampling_matches_reference(golden_sampling, cfg1_graph):
    g = golden_sampling
    prefixes = batch_prefixes(g)
    assert len(prefixes) >= 20
    for p in prefixes:
        graph = _graph_for(p, g) or cfg1_graph
        seed, epoch, bid = (int(x) for x in g[f"{p}/key"])
        mask_name = str(g[f"{p}/mask_name"])
        mask = g[mask_name] if mask_name else None
        targets, layers, digest, hits = golden_batch(g, p)
        mb = osamp.build_minibatch(graph.row_offsets, graph.col_indices, graph.features,
                                   graph.labels, targets, tuple(g[f"{p}/fanouts"]), seed=seed,
                                   epoch=epoch, batch_id=bid, cached_mask=mask)
        for l, ref in enumerate(layers):
            blk = mb.layers[l]
            for k in ("rows", "cols", "values", "src_ids", "dst_ids"):
                assert np.array_equal(getattr(blk, k), ref[k]), (p, l, k)
        assert mb.digest() == digest, p
        assert [mb.cache_hits, mb.cache_misses] == list(hits)


def test_cfg1_graph_is_the_golden_graph(golden_sampling, cfg1_graph):
    import hashlib
    h = hashlib.sha256(cfg1_graph.row_offsets.tobytes()
                       + cfg1_graph.col_indices.astype(np.int64).tobytes()).digest()
    assert h == bytes(golden_sampling["cfg1/row_offsets_sha"])


def _oracle_batch(golden_s, graph, targets, fanouts, key, mask):
    return osamp.build_minibatch(graph.row_offsets, graph.col_indices, graph.features,
                                 graph.labels, targets, fanouts, seed=key[0], epoch=key[1],
                                 batch_id=key[2], cached_mask=mask)


@pytest.mark.parametrize("tag", ["2l", "3l"])
def test_oracle_numerics_match_reference(golden_nn, golden_sampling, tag):
    gn, gs = golden_nn, golden_sampling
    graph = make_g2(gs)
    fanouts = tuple(gn[f"{tag}/fanouts"])
    hidden = int(gn[f"{tag}/hidden"][0])
    model = onn.init_model(16, hidden, 5, num_layers=len(fanouts), seed=7, learning_rate=0.01)
    for step in range(3):
        p = f"{tag}/s{step}"
        for l, w in enumerate(model.weights):
            assert np.array_equal(w, gn[f"{p}/w_before{l}"])
        mb = _oracle_batch(gs, graph, gn[f"{p}/targets"], fanouts, (4, 0, step), gs["g2/mask10"])
        logits, cache = onn.sage_forward(mb.layers, mb.features, model.weights)
        # same NumPy kernels in the same order: bit-identical
        assert np.array_equal(logits, gn[f"{p}/logits"])
        loss, dl = onn.batch_loss(logits, mb.target_labels)
        assert loss == float(gn[f"{p}/loss"][0])
        assert np.array_equal(dl, gn[f"{p}/dlogits"])
        grads = onn.backward(mb.layers, model.weights, cache, dl)
        for l, gr in enumerate(grads):
            assert np.array_equal(gr, gn[f"{p}/grad{l}"])
        onn.adam_step(model, grads)
        for l in range(len(model.weights)):
            assert np.array_equal(model.weights[l], gn[f"{p}/w_after{l}"])
            assert np.array_equal(model.m[l], gn[f"{p}/m_after{l}"])
            assert np.array_equal(model.v[l], gn[f"{p}/v_after{l}"])


def test_oracle_sgd_matches_reference(golden_nn):
    model = onn.init_model(16, 32, 5, num_layers=2, seed=7, learning_rate=0.05)
    onn.sgd_step(model, [golden_nn["2l/s0/grad0"], golden_nn["2l/s0/grad1"]])
    for l in range(2):
        assert np.array_equal(model.weights[l], golden_nn[f"sgd/w_after{l}"])


def test_oracle_gather_matches_reference(golden_cache, golden_sampling):
    gc = golden_cache
    graph = make_g2(golden_sampling)
    cached_ids = gc["cached_ids"]
    feats_cache = graph.features[cached_ids].copy()
    out = ocache.gather_features(cached_ids, gc["mask"], feats_cache, graph.features, gc["ids"])
    assert np.array_equal(out, gc["gather"])
    hits, misses = ocache.lookup(gc["mask"], gc["ids"])
    assert np.array_equal(hits, gc["hits"]) and np.array_equal(misses, gc["misses"])
    marked = ocache.gather_features(cached_ids, gc["mask"], feats_cache + 100.0, graph.features,
                                    gc["ids"])
    assert np.array_equal(marked, gc["gather_marked"])


def test_oracle_plan_epoch_matches_reference(golden_runtime, golden_sampling):
    rt = golden_runtime
    tm = golden_sampling["g2/train_mask"]
    for G, B in ((1, 256), (2, 256), (3, 200), (4, 128)):
        per_dev, expected = oracom.plan_epoch(tm, G, B, seed=9, epoch=3)
        assert expected == rt[f"plan/G{G}_B{B}/expected"].tolist()
        for d in range(G):
            assert [b for _, b, _ in per_dev[d]] == rt[f"plan/G{G}_B{B}/d{d}/bids"].tolist()
            assert np.array_equal(np.concatenate([t for _, _, t in per_dev[d]]),
                                  rt[f"plan/G{G}_B{B}/d{d}/targets"])


def test_oracle_sync_period_matches_reference(golden_runtime):
    for V, E, G, k, want in golden_runtime["sync_periods"]:
        assert oracom.compute_sync_period(int(V), int(E), int(G), float(k)) == int(want)


@pytest.mark.parametrize("name", ["1dev_adam", "2dev_adam", "2dev_sgd_p3", "3dev_adam_p2"])
def test_oracle_run_epoch_matches_reference(golden_runtime, golden_sampling, name):
    rt, gs = golden_runtime, golden_sampling
    G, B, seed, P = (int(x) for x in rt[f"epoch/{name}/config"])
    graph = make_g2(gs)
    masks = {"2dev_adam": gs["g2/mask10"], "3dev_adam_p2": gs["g2/mask1"]}
    gdict = dict(row_offsets=graph.row_offsets, col_indices=graph.col_indices,
                 features=graph.features, labels=graph.labels, train_mask=rt["epoch/train_mask"])
    opt = "sgd" if "sgd" in name else "adam"
    base = onn.init_model(16, 16, 5, num_layers=2, seed=5, learning_rate=0.01)
    models = [base.copy() for _ in range(G)]
    losses, traces = oracom.run_epoch_serial(gdict, models, fanouts=(4, 3), batch_size=B,
                                             seed=seed, epoch=1, optimizer=opt, sync_period=P,
                                             cached_mask=masks.get(name), capture_weights=True)
    bids = rt[f"epoch/{name}/loss_bids"].tolist()
    assert sorted(losses) == bids
    # serial zero-delay schedule: the f64 mean of the same f32 grads -> identical
    got = np.array([losses[b] for b in bids])
    assert np.array_equal(got, rt[f"epoch/{name}/losses"])
    for l in range(2):
        assert np.array_equal(models[0].weights[l], rt[f"epoch/{name}/w{l}"])
        assert np.array_equal(models[0].m[l], rt[f"epoch/{name}/m{l}"])
        assert np.array_equal(models[0].v[l], rt[f"epoch/{name}/v{l}"])
    assert [k for k, _ in traces[0]] == rt[f"epoch/{name}/trace_windows"].tolist()
