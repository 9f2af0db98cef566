"""Golden fixtures of the per-epoch functions around the hot path, made by
running the REFERENCE itself (build container only: needs /root/reference).

    python tests/golden/make_golden_epoch.py

* evaluation: ``mqpipe.nn.full_forward`` (nn.py:218-250) and the driver's
  ``evaluate`` (bench.py:82-87) on the G2 power-law graph (stored self loops)
  and the g8 edge-case graph, 2- and 3-layer SAGE models, before and after a
  few training steps;
* cache refresh: ``cache_probs_degree`` (cache.py:41-48), ``cache_probs_walk``
  (cache.py:51-76) and ``refresh_cache`` (cache.py:79-108) driven through the
  refresh injected-draw contract (``oracle.philox.RefreshRng``: ``random(n)``
  and WOR ``choice`` from reserved Philox row streams), including a
  zero-probability shortfall case.

Output: ``epoch.npz`` next to this script.
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(HERE))
sys.path.insert(0, str(HERE.parent))
sys.path.insert(0, "/root/reference/pkg/src")

import mqpipe  # noqa: E402
from mqpipe import bench as rbench  # noqa: E402
from mqpipe import cache as rcache  # noqa: E402
from mqpipe import nn as rnn  # noqa: E402

from make_golden import BatchKey, g8, synth_ref, with_self_loops  # noqa: E402
from conftest import EDGES_8 as G8_EDGES  # noqa: E402
from oracle.philox import RefreshRng  # noqa: E402


def main():
    out = {}
    G2 = with_self_loops(synth_ref(2000, 20000, 16, 5, seed=11))
    G8 = g8()
    for gname, G in (("g2", G2), ("g8", G8)):
        out[f"{gname}/row_offsets"] = G.row_offsets
        out[f"{gname}/col_indices"] = G.col_indices
        out[f"{gname}/features"] = G.features
        out[f"{gname}/labels"] = G.labels
        out[f"{gname}/train_mask"] = G.train_mask
        out[f"{gname}/val_mask"] = G.val_mask
        out[f"{gname}/test_mask"] = G.test_mask

    # ---- evaluation
    for tag, G, hidden, layers, fo in (("g2_2l", G2, 32, 2, (10, 5)), ("g2_3l", G2, 24, 3, (3, 3, 2)),
                                       ("g8_2l", G8, 4, 2, (2, 2))):
        state = rnn.init_model(G.feature_dim, hidden, G.num_classes, num_layers=layers,
                               arch="sage", seed=7, learning_rate=0.01)
        params = mqpipe.SamplerParams(method="sage", fanout=fo, num_layers=layers)
        for phase in range(2):
            if phase == 1:  # a few Adam steps so the logits are not the init's
                tr = np.flatnonzero(G.train_mask)
                for step in range(3):
                    tg = tr[(step * 64) % max(tr.size, 1):][:64]
                    if tg.size == 0:
                        tg = tr[:64]
                    mb = mqpipe.build_minibatch(G, tg, params, BatchKey(5, 0, step),
                                                batch_id=step, epoch=0)
                    _, grads = rnn.loss_and_grads(mb, state)[:2]
                    rnn.adam_step(state, grads)
            p = f"eval/{tag}/p{phase}"
            for l, w in enumerate(state.weights):
                out[f"{p}/w{l}"] = w.copy()
            out[f"{p}/logits"] = rnn.full_forward(G, state)
            out[f"{p}/val_acc"] = np.array([rbench.evaluate(G, state, G.val_mask)])
            out[f"{p}/test_acc"] = np.array([rbench.evaluate(G, state, G.test_mask)])
        out[f"eval/{tag}/graph"] = np.array(tag[:2])

    # ---- cache refresh
    out["refresh/g2/degree_probs"] = rcache.cache_probs_degree(G2)
    for fo, steps in ((5, 2), (10, 3)):
        out[f"refresh/g2/walk_probs_f{fo}_s{steps}"] = rcache.cache_probs_walk(G2, fo, steps)
    # a small training set leaves unreachable nodes at probability zero
    small = G2.train_mask.copy()
    small[np.flatnonzero(small)[3:]] = False
    Gs = mqpipe.GraphCSR(num_nodes=G2.num_nodes, row_offsets=G2.row_offsets,
                         col_indices=G2.col_indices, features=G2.features, labels=G2.labels,
                         num_classes=G2.num_classes, train_mask=small, val_mask=G2.val_mask,
                         test_mask=G2.test_mask)
    out["refresh/g2small/train_mask"] = small
    out["refresh/g2small/walk_probs_f2_s1"] = rcache.cache_probs_walk(Gs, 2, 1)
    cases = [("deg_1pct", "refresh/g2/degree_probs", 0.01, 3, 0),
             ("deg_10pct", "refresh/g2/degree_probs", 0.10, 3, 1),
             ("walk_5pct", "refresh/g2/walk_probs_f5_s2", 0.05, 9, 2),
             ("walk_30pct", "refresh/g2/walk_probs_f10_s3", 0.30, 1, 0),
             ("short_50pct", "refresh/g2small/walk_probs_f2_s1", 0.50, 4, 7)]
    for name, probs_key, frac, seed, epoch in cases:
        probs = out[probs_key]
        c = rcache.refresh_cache(G2, probs, frac, RefreshRng(seed, epoch))
        p = f"refresh/case/{name}"
        out[f"{p}/probs_key"] = np.array(probs_key)
        out[f"{p}/params"] = np.array([frac, seed, epoch], dtype=np.float64)
        out[f"{p}/cached_ids"] = c.cached_ids
        out[f"{p}/positive"] = np.array([int(np.count_nonzero(probs > 0))])
    # ---- ingest: the reference's build_csr (graph.py:94-139) and its MQG1 container
    from mqpipe import graph as rgraph
    rng = np.random.default_rng(31)
    n = 1000
    e_rand = rng.integers(0, n, size=(20000, 2))
    e_rand = np.concatenate([e_rand, e_rand[:500], np.stack([np.arange(0, n, 9)] * 2, 1)])
    rng.shuffle(e_rand)
    hub = np.stack([np.zeros(3000, np.int64), rng.integers(0, 5000, 3000)], 1)
    e_hub = np.concatenate([hub, hub[:, ::-1], rng.integers(0, 5000, size=(4000, 2))])
    for name, edges, nn_ in (("g8", np.asarray(G8_EDGES), 8), ("rand", e_rand, n),
                             ("hub", e_hub, 5000)):
        g = rgraph.build_csr(edges, nn_)
        out[f"ingest/{name}/edges"] = np.asarray(edges, dtype=np.int64)
        out[f"ingest/{name}/n"] = np.array([nn_])
        out[f"ingest/{name}/row_offsets"] = g.row_offsets
        out[f"ingest/{name}/col_indices"] = g.col_indices
        out[f"ingest/{name}/features"] = g.features
    out["ingest/mqg1"] = np.frombuffer(rgraph.serialize(G2), dtype=np.uint8).copy()

    # ---- queue sizing formulas (autotune.py:29-34, 112-141)
    from mqpipe import autotune as rauto
    caps, qs, sl = [], [], []
    for total, peak, mb in ((24 * 2**30, 10 * 2**30, 2**28), (100, 40, 10), (10**9, 5 * 10**8, 7),
                            (50, 40, 10)):
        try:
            caps.append([total, peak, mb, rauto.compute_cap(total, peak, mb)])
        except rauto.AutotuneError:
            caps.append([total, peak, mb, -1])
    for prep, comp, cap in ((7.0, 2.0, 10), (0.5, 3.0, 8), (30.0, 1.0, 6), (1.0, 1.0, 1)):
        qs.append([prep, comp, cap, rauto.compute_queue_size(prep, comp, cap)])
    for n in (5, 59, 60, 100, 41):
        s_ = rauto.steady_slice(n)
        sl.append([n, s_.start, s_.stop])
    out["autotune/cap"] = np.array(caps, dtype=np.float64)
    out["autotune/queue"] = np.array(qs, dtype=np.float64)
    out["autotune/steady"] = np.array(sl, dtype=np.int64)
    np.savez_compressed(HERE / "epoch.npz", **out)
    print("epoch.npz", os.path.getsize(HERE / "epoch.npz"))


if __name__ == "__main__":
    main()
