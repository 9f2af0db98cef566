"""Generate the golden fixtures by running the REFERENCE itself.

Run in the build container (the only place ``/root/reference`` exists):

    python tests/golden/make_golden.py

It imports ``mqpipe`` from ``/root/reference/pkg/src`` and drives the
reference's own functions under the injected Philox draw contract
(SURVEY.md §8c):

* ``RowIndexedRng`` — a duck-typed ``rng`` whose k-th ``choice`` call draws
  from the Philox stream of the k-th row that calls ``choice`` in
  ``node_wise_block`` (rows with more non-loop neighbours than the fanout,
  ``samplers.py:163-177``); the partial Fisher-Yates selection is the contract.
* ``sample_node_wise`` is replaced by a per-hop-fanout loop over the
  reference's own ``node_wise_block`` (hop index = depth from the seeds), and
  ``runtime.batch_rng`` by a key carrying (seed, epoch, batch_id).

Everything else (block construction, relabel, values, digests, gather,
forward/backward/loss/Adam/SGD, plan_epoch, run_epoch) is the unmodified
reference.  Outputs: ``philox_kat.json``, ``sampling.npz``, ``nn.npz``,
``cache.npz``, ``runtime.npz`` next to this script.
"""

from __future__ import annotations

import json
import os
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, "/root/reference/pkg/src")

import mqpipe  # noqa: E402
from mqpipe import cache as rcache  # noqa: E402
from mqpipe import nn as rnn  # noqa: E402
from mqpipe import racom as rracom  # noqa: E402
from mqpipe import runtime as rruntime  # noqa: E402
from mqpipe import samplers as rsamplers  # noqa: E402

from oracle.philox import draws, fisher_yates_positions, philox4x32_10  # noqa: E402
from paper_2601_04707_b200.synth import generate_numpy, keys_to_csr  # noqa: E402

# ------------------------------------------------------------------ the shim


class BatchKey:
    def __init__(self, seed, epoch, batch_id):
        self.seed, self.epoch, self.batch_id = seed, epoch, batch_id


class RowIndexedRng:
    def __init__(self, key: BatchKey, hop: int, rows):
        self.key, self.hop, self.rows, self.k = key, hop, list(rows), 0

    def choice(self, a, size, replace=False):
        assert not replace
        row = self.rows[self.k]
        self.k += 1
        x = draws(self.key.seed, self.key.epoch, self.key.batch_id, self.hop, row, size)
        a = np.asarray(a)
        return a[fisher_yates_positions(x, a.size, size)]


def per_hop_sample_node_wise(g, targets, fanout, layers, rng, arch="gcn", cached_mask=None):
    dst = np.asarray(targets, dtype=np.int64)
    if dst.size == 0:
        raise rsamplers.SamplingError("empty target set")
    fanouts = tuple(fanout) if isinstance(fanout, (tuple, list)) else (fanout,) * layers
    blocks = []
    for hop, f in enumerate(fanouts):
        rows = []
        for r, v in enumerate(dst.tolist()):
            nb = g.out_neighbors(v)
            if int(np.count_nonzero(nb != v)) > f:
                rows.append(r)
        shim = RowIndexedRng(rng, hop, rows)
        blk = rsamplers.node_wise_block(g, dst, f, shim, arch=arch, cached_mask=cached_mask)
        assert shim.k == len(rows), "choice-call count mismatch"
        blocks.append(blk)
        dst = blk.src_ids
    blocks.reverse()
    return blocks


rsamplers.sample_node_wise = per_hop_sample_node_wise
rruntime.batch_rng = lambda config, epoch, batch_id: BatchKey(config.seed, epoch, batch_id)

# ------------------------------------------------------------------ graphs
EDGES_8 = [
    (0, 1), (1, 0), (0, 2), (2, 0), (1, 2), (2, 1),
    (2, 3), (3, 2), (3, 3), (3, 4), (4, 3), (4, 5), (5, 4),
    (5, 6), (6, 5), (6, 7), (7, 6), (7, 0), (0, 7),
    (1, 5), (5, 1), (2, 6), (6, 2),
]


def g8():
    rng = np.random.default_rng(42)
    feats = rng.standard_normal((8, 3)).astype(np.float32)
    labels = np.array([0, 1, 0, 1, 0, 1, 0, 1], dtype=np.int32)
    g = mqpipe.build_csr(EDGES_8, 8, features=feats, labels=labels, num_classes=2)
    return mqpipe.split_masks(g, ratios=(0.5, 0.25, 0.25), seed=0)


def synth_ref(n, arcs, d, c, seed, train=0.66):
    """The synthetic graph rebuilt through the reference's own build_csr."""
    sg = generate_numpy(n, arcs, d, c, train=train, seed=seed)
    src = np.repeat(np.arange(n), np.diff(sg.row_offsets))
    edges = np.stack([src, sg.col_indices], axis=1)
    g = mqpipe.build_csr(edges, n, features=sg.features, labels=sg.labels, num_classes=c)
    assert np.array_equal(g.row_offsets, sg.row_offsets)
    assert np.array_equal(g.col_indices, sg.col_indices)
    return mqpipe.GraphCSR(num_nodes=n, row_offsets=g.row_offsets, col_indices=g.col_indices,
                           features=g.features, labels=g.labels, num_classes=c,
                           train_mask=sg.train_mask, val_mask=sg.val_mask,
                           test_mask=sg.test_mask)


def with_self_loops(g, every=7):
    """Add stored self loops on every `every`-th node (reference keeps them)."""
    n = g.num_nodes
    src = np.repeat(np.arange(n), np.diff(g.row_offsets))
    extra = np.arange(0, n, every)
    edges = np.concatenate([np.stack([src, g.col_indices], 1), np.stack([extra, extra], 1)])
    h = mqpipe.build_csr(edges, n, features=g.features, labels=g.labels,
                         num_classes=g.num_classes)
    return mqpipe.GraphCSR(num_nodes=n, row_offsets=h.row_offsets, col_indices=h.col_indices,
                           features=h.features, labels=h.labels, num_classes=g.num_classes,
                           train_mask=g.train_mask, val_mask=g.val_mask, test_mask=g.test_mask)


def degree_cache(g, fraction, seed):
    rng = np.random.default_rng(seed)
    return rcache.refresh_cache(g, rcache.cache_probs_degree(g), fraction, rng)


# ------------------------------------------------------------------ helpers
def store_batch(out, prefix, mb, key, mask_name):
    out[f"{prefix}/key"] = np.array([key.seed, key.epoch, key.batch_id], dtype=np.int64)
    out[f"{prefix}/mask_name"] = np.array(mask_name)
    out[f"{prefix}/targets"] = mb.target_ids
    out[f"{prefix}/labels"] = mb.target_labels
    out[f"{prefix}/digest"] = np.frombuffer(bytes.fromhex(mb.digest()), dtype=np.uint8)
    out[f"{prefix}/hits"] = np.array([mb.cache_hits, mb.cache_misses])
    for l, blk in enumerate(mb.layers):
        for k in ("rows", "cols", "values", "src_ids", "dst_ids"):
            out[f"{prefix}/L{l}/{k}"] = getattr(blk, k)


def main():
    # ---- Philox KAT + stream/selection vectors
    # Random123 published known-answer vectors for philox4x32_10 (kat_vectors)
    kat = [{"ctr": [0, 0, 0, 0], "key": [0, 0],
            "out": [0x6627e8d5, 0xe169c58d, 0xbc57ac4c, 0x9b00dbd8]},
           {"ctr": [0xFFFFFFFF] * 4, "key": [0xFFFFFFFF] * 2,
            "out": [0x408f276d, 0x41c83b0e, 0xa20bc7c6, 0x6d5451fd]},
           {"ctr": [0x243f6a88, 0x85a308d3, 0x13198a2e, 0x03707344],
            "key": [0xa4093822, 0x299f31d0],
            "out": [0xd16cfe09, 0x94fdcceb, 0x5001e420, 0x24126ea1]}]
    for v in kat:
        assert philox4x32_10(np.array(v["ctr"]), np.array(v["key"])).tolist() == v["out"]
    streams = []
    for (seed, epoch, batch, hop, row, n, k) in [(0, 0, 0, 0, 0, 100, 10), (7, 3, 11, 1, 5, 17, 5),
                                                (2**40 + 5, 9, 123, 2, 999, 1_000_000, 15),
                                                (1, 1, 1, 1, 1, 32, 32), (5, 0, 2, 0, 3, 6, 5)]:
        x = draws(seed, epoch, batch, hop, row, k)
        streams.append({"seed": seed, "epoch": epoch, "batch": batch, "hop": hop, "row": row,
                        "n": n, "k": k, "draws": x.tolist(),
                        "positions": fisher_yates_positions(x, n, k)})
    (HERE / "philox_kat.json").write_text(json.dumps({"kat": kat, "streams": streams}, indent=1))

    samp = {}
    # ---- g8 (reference conftest fixture): edge cases incl. stored self loop
    G8 = g8()
    cases8 = [("g8_f2", [0, 3], (2,), None),
              ("g8_all_f1", list(range(8)), (1,), None),
              ("g8_all_f1_cached", list(range(8)), (1,), [1, 2]),
              ("g8_dup", [0, 0, 3, 3, 5], (2, 2), None),
              ("g8_cached4", list(range(8)), (3, 2), [0, 1, 2, 3]),
              ("g8_bigfanout", list(range(8)), (8, 8), None)]
    for name, tg, fo, cached in cases8:
        mask = None
        if cached is not None:
            mask = np.zeros(8, dtype=bool)
            mask[cached] = True
            samp[f"{name}/mask"] = mask
        params = mqpipe.SamplerParams(method="sage", fanout=fo, num_layers=len(fo))
        key = BatchKey(3, 1, 4)
        mb = mqpipe.build_minibatch(G8, np.array(tg), params, key, batch_id=4,
                                    epoch=1, cached_mask=mask)
        store_batch(samp, name, mb, key, f"{name}/mask" if cached is not None else "")
        samp[f"{name}/fanouts"] = np.array(fo)
    # ---- synthetic power-law graph with stored self loops, several caches
    G2 = with_self_loops(synth_ref(2000, 20000, 16, 5, seed=11))
    samp["g2/row_offsets"] = G2.row_offsets
    samp["g2/col_indices"] = G2.col_indices.astype(np.int32)
    samp["g2/features"] = G2.features
    samp["g2/labels"] = G2.labels
    samp["g2/train_mask"] = G2.train_mask
    c1 = degree_cache(G2, 0.01, 5)
    c10 = degree_cache(G2, 0.10, 6)
    samp["g2/mask1"] = c1.cached_mask
    samp["g2/mask10"] = c10.cached_mask
    rng = np.random.default_rng(0)
    for cname, cache in (("nocache", None), ("c1", c1), ("c10", c10)):
        for fo in ((10, 5), (3, 3, 2), (1,)):
            for b in range(2):
                tg = rng.choice(np.flatnonzero(G2.train_mask), size=256, replace=False)
                params = mqpipe.SamplerParams(method="sage", fanout=fo, num_layers=len(fo))
                mask = cache.cached_mask if cache is not None else None
                name = f"g2_{cname}_{'x'.join(map(str, fo))}_b{b}"
                key = BatchKey(17, 2, 30 + b)
                mb = mqpipe.build_minibatch(G2, tg, params, key,
                                            batch_id=30 + b, epoch=2, cached_mask=mask)
                store_batch(samp, name, mb, key,
                            {"nocache": "", "c1": "g2/mask1", "c10": "g2/mask10"}[cname])
                samp[f"{name}/fanouts"] = np.array(fo)
    # ---- cfg1 shape (configs[0]): first two batches of epoch 0, 1% degree cache
    G1 = synth_ref(10_000, 100_000, 64, 4, seed=0)
    c_cfg1 = degree_cache(G1, 0.01, 3)
    samp["cfg1/mask"] = c_cfg1.cached_mask
    samp["cfg1/row_offsets_sha"] = np.frombuffer(
        __import__("hashlib").sha256(G1.row_offsets.tobytes() + G1.col_indices.tobytes()).digest(),
        dtype=np.uint8)
    cfg = rruntime.PipelineConfig(num_devices=1, batch_size=1024,
                                  sampler=mqpipe.SamplerParams(method="sage", fanout=(10, 5),
                                                               num_layers=2), seed=0)
    per_dev, _ = rruntime.plan_epoch(G1, cfg, 0)
    for w, bid, tg in per_dev[0][:2]:
        key = BatchKey(0, 0, bid)
        mb = mqpipe.build_minibatch(G1, tg, cfg.sampler, key, batch_id=bid, epoch=0,
                                    cached_mask=c_cfg1.cached_mask)
        store_batch(samp, f"cfg1_b{bid}", mb, key, "cfg1/mask")
        samp[f"cfg1_b{bid}/fanouts"] = np.array((10, 5))
    np.savez_compressed(HERE / "sampling.npz", **samp)

    # ---- numerics on G2 batches (float32 training dtype)
    nn_out = {}
    for tag, fo, hidden in (("2l", (10, 5), 32), ("3l", (3, 3, 2), 24)):
        params = mqpipe.SamplerParams(method="sage", fanout=fo, num_layers=len(fo))
        state = rnn.init_model(16, hidden, 5, num_layers=len(fo), arch="sage", seed=7,
                               learning_rate=0.01)
        for step in range(3):
            tg = np.flatnonzero(G2.train_mask)[step * 200:(step + 1) * 200]
            mb = mqpipe.build_minibatch(G2, tg, params, BatchKey(4, 0, step), batch_id=step,
                                        epoch=0, cached_mask=c10.cached_mask)
            logits, cache = rnn.forward(mb, state, return_cache=True)
            loss, dl = rnn.batch_loss(logits, mb.target_labels)
            grads = rnn.backward(mb, state, cache, dl)
            p = f"{tag}/s{step}"
            nn_out[f"{p}/targets"] = tg
            for l, w in enumerate(state.weights):
                nn_out[f"{p}/w_before{l}"] = w.copy()
            nn_out[f"{p}/logits"] = logits
            nn_out[f"{p}/loss"] = np.array([loss])
            nn_out[f"{p}/dlogits"] = dl
            for l, (h, both) in enumerate(cache["inputs"]):
                nn_out[f"{p}/agg{l}"] = both[:, :h.shape[1]]
            for l, g in enumerate(grads):
                nn_out[f"{p}/grad{l}"] = g
            rnn.adam_step(state, grads)
            for l in range(len(state.weights)):
                nn_out[f"{p}/w_after{l}"] = state.weights[l].copy()
                nn_out[f"{p}/m_after{l}"] = state.m[l].copy()
                nn_out[f"{p}/v_after{l}"] = state.v[l].copy()
        nn_out[f"{tag}/fanouts"] = np.array(fo)
        nn_out[f"{tag}/hidden"] = np.array([hidden])
    # SGD closed form on the same grads
    st = rnn.init_model(16, 32, 5, num_layers=2, arch="sage", seed=7, learning_rate=0.05)
    grads = [nn_out["2l/s0/grad0"], nn_out["2l/s0/grad1"]]
    rnn.sgd_step(st, grads)
    for l in range(2):
        nn_out[f"sgd/w_after{l}"] = st.weights[l].copy()
    np.savez_compressed(HERE / "nn.npz", **nn_out)

    # ---- gather / lookup (cache.py:111-134) incl. hits routed to the cache copy
    cache_out = {}
    c = degree_cache(G2, 0.10, 9)
    ids = np.concatenate([c.cached_ids[:5], np.arange(0, 2000, 97), c.cached_ids[:3],
                          c.cached_ids[:1]]).astype(np.int64)
    cache_out["ids"] = ids
    cache_out["mask"] = c.cached_mask
    cache_out["cached_ids"] = c.cached_ids
    cache_out["gather"] = rcache.gather_features(c, G2, ids)
    hits, misses = rcache.lookup(c, ids)
    cache_out["hits"] = hits
    cache_out["misses"] = misses
    c.cached_features += 100.0
    cache_out["gather_marked"] = rcache.gather_features(c, G2, ids)
    np.savez_compressed(HERE / "cache.npz", **cache_out)

    # ---- plan_epoch, sync period, run_epoch (serial deterministic schedule)
    rt = {}
    for G, B in ((1, 256), (2, 256), (3, 200), (4, 128)):
        cfg = rruntime.PipelineConfig(num_devices=G, batch_size=B, seed=9)
        per_dev, expected = rruntime.plan_epoch(G2, cfg, 3)
        rt[f"plan/G{G}_B{B}/expected"] = np.array(expected)
        for d in range(G):
            rt[f"plan/G{G}_B{B}/d{d}/bids"] = np.array([b for _, b, _ in per_dev[d]])
            rt[f"plan/G{G}_B{B}/d{d}/targets"] = np.concatenate([t for _, _, t in per_dev[d]])
    periods = []
    for (V, E, G, k) in [(10_000, 100_000, 1, 1.0), (232_965, 114_000_000, 8, 1.0),
                         (2_449_029, 62_000_000, 4, 1.0), (100, 0, 2, 1.0), (1_000_000, 10, 2, 3.0),
                         (50, 40, 1, 2.5)]:
        import warnings
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            periods.append([V, E, G, k, rracom.compute_sync_period(V, E, G, k)])
    rt["sync_periods"] = np.array(periods, dtype=np.float64)
    Gs = mqpipe.split_masks(G2, ratios=(0.3, 0.1, 0.1), seed=2)
    for name, G, opt, P, cached in (("1dev_adam", 1, "adam", 1, None),
                                    ("2dev_adam", 2, "adam", 1, c10),
                                    ("2dev_sgd_p3", 2, "sgd", 3, None),
                                    ("3dev_adam_p2", 3, "adam", 2, c1)):
        cfg = rruntime.PipelineConfig(
            num_devices=G, batch_size=64,
            sampler=mqpipe.SamplerParams(method="sage", fanout=(4, 3), num_layers=2),
            optimizer=opt, sync_period=P, deterministic=True, seed=5, capture_weights=True)
        base = rnn.init_model(16, 16, 5, num_layers=2, arch="sage", seed=5, learning_rate=0.01)
        reps = [base.copy() for _ in range(G)]
        stats, _ = rruntime.run_epoch(Gs, cached, reps, cfg, epoch=1)
        rt[f"epoch/{name}/loss_bids"] = np.array(sorted(stats.losses))
        rt[f"epoch/{name}/losses"] = np.array([stats.losses[b] for b in sorted(stats.losses)])
        rt[f"epoch/{name}/sync_count"] = np.array([stats.sync_count, stats.epoch_sync])
        rt[f"epoch/{name}/hits"] = np.array([stats.cache_hits, stats.cache_misses])
        for l in range(2):
            rt[f"epoch/{name}/w{l}"] = reps[0].weights[l]
            rt[f"epoch/{name}/m{l}"] = reps[0].m[l]
            rt[f"epoch/{name}/v{l}"] = reps[0].v[l]
        wt = stats.weight_traces[0]
        rt[f"epoch/{name}/trace_windows"] = np.array([k for k, _ in wt])
        rt[f"epoch/{name}/trace_w0_first"] = wt[0][1][0]
        rt[f"epoch/{name}/config"] = np.array([G, 64, 5, P])
    rt["epoch/train_mask"] = Gs.train_mask
    np.savez_compressed(HERE / "runtime.npz", **rt)
    for f in sorted(HERE.glob("*.npz")) + [HERE / "philox_kat.json"]:
        print(f.name, os.path.getsize(f))


if __name__ == "__main__":
    main()
