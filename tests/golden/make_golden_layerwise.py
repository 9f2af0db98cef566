"""Golden fixtures for the layer-wise samplers and the GCN block arm, made by
the REFERENCE itself.

Run in the build container (the only place ``/root/reference`` exists):

    python tests/golden/make_golden_layerwise.py

The reference's own ``build_minibatch`` / ``sample_ladies`` /
``sample_fastgcn`` / ``ladies_probs`` / ``flat_probs`` / ``fastgcn_probs`` /
``debias_coefficients`` run unmodified; the only injected piece is the batch
``rng``: ``oracle.layerwise.LayerRng`` (one public call per layer, draws from
the layer's Philox stream; ``choice(.., replace=True, p)`` is NumPy's
published algorithm over those uniforms).  The GCN node-wise arm goes through
the same per-row Philox shim as ``make_golden.py``.  Output:
``layerwise.npz`` next to this script.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))
import make_golden as mg  # noqa: E402  (also installs the node-wise shim)

mqpipe, rsamplers = mg.mqpipe, mg.rsamplers
from oracle.layerwise import LayerRng  # noqa: E402

KEY = (5, 2, 9)   # seed, epoch, batch_id


def g9_isolated():
    """g8 plus an isolated node 8 (a zero-out-degree target gets dropped)."""
    rng = np.random.default_rng(42)
    feats = rng.standard_normal((9, 3)).astype(np.float32)
    labels = np.array([0, 1, 0, 1, 0, 1, 0, 1, 0], dtype=np.int32)
    return mqpipe.build_csr(mg.EDGES_8, 9, features=feats, labels=labels, num_classes=2)


def store(out, prefix, mb, params):
    out[f"{prefix}/key"] = np.array([KEY[0], KEY[1], KEY[2]], dtype=np.int64)
    out[f"{prefix}/params"] = np.array([params.nodes_per_layer, params.num_layers,
                                        int(params.flat), int(params.debias),
                                        int(params.replace)], dtype=np.int64)
    out[f"{prefix}/method"] = np.array(params.method)
    out[f"{prefix}/target_ids"] = mb.target_ids
    out[f"{prefix}/labels"] = mb.target_labels
    out[f"{prefix}/dropped"] = np.array(mb.dropped_targets)
    out[f"{prefix}/digest"] = np.frombuffer(bytes.fromhex(mb.digest()), dtype=np.uint8)
    out[f"{prefix}/features"] = mb.features
    for l, blk in enumerate(mb.layers):
        for k in ("rows", "cols", "values", "effective_values", "src_ids", "dst_ids"):
            out[f"{prefix}/L{l}/{k}"] = getattr(blk, k)
        if blk.sample_probs is not None:
            out[f"{prefix}/L{l}/sample_probs"] = blk.sample_probs


def main():
    out = {}
    G8 = mg.g8()
    G9 = g9_isolated()
    G2 = mg.with_self_loops(mg.synth_ref(2000, 20000, 16, 5, seed=11))
    graphs = {"g8": G8, "g9": G9, "g2": G2}
    for name, g in graphs.items():
        out[f"graph/{name}/row_offsets"] = g.row_offsets
        out[f"graph/{name}/col_indices"] = g.col_indices
        out[f"graph/{name}/a_hat_degrees"] = g.a_hat_degrees

    rng = np.random.default_rng(3)
    t2 = rng.choice(2000, size=96, replace=False)
    cases = [
        # name, graph, targets, method, budget, layers, flat, debias, replace
        ("g8_ladies", "g8", [0, 3, 5], "ladies", 3, 2, False, False, False),
        ("g8_ladies_flat", "g8", [0, 3, 5], "ladies", 3, 2, True, False, False),
        ("g8_ladies_debias", "g8", [0, 3, 5], "ladies", 3, 2, False, True, False),
        ("g8_ladies_replace", "g8", [0, 3, 5], "ladies", 4, 2, False, False, True),
        ("g8_ladies_all", "g8", list(range(8)), "ladies", 8, 2, False, False, False),
        ("g9_ladies_drop", "g9", [8, 1, 8, 6], "ladies", 3, 1, False, False, False),
        ("g8_fastgcn", "g8", [0, 3, 5], "fastgcn", 4, 2, False, False, False),
        ("g8_fastgcn_flat", "g8", [0, 3, 5], "fastgcn", 4, 2, True, False, False),
        ("g8_fastgcn_debias", "g8", [0, 3, 5], "fastgcn", 3, 2, False, True, False),
        ("g2_ladies", "g2", t2, "ladies", 64, 2, False, False, False),
        ("g2_ladies_flat_debias", "g2", t2, "ladies", 64, 2, True, True, False),
        ("g2_ladies_replace", "g2", t2, "ladies", 64, 3, False, False, True),
        ("g2_ladies_big", "g2", t2, "ladies", 1500, 2, False, False, False),
        ("g2_fastgcn", "g2", t2, "fastgcn", 128, 2, False, False, False),
        ("g2_fastgcn_flat_debias", "g2", t2, "fastgcn", 128, 2, True, True, False),
    ]
    names = []
    for name, gname, tg, method, budget, layers, flat, debias, replace in cases:
        g = graphs[gname]
        params = mqpipe.SamplerParams(method=method, nodes_per_layer=budget, num_layers=layers,
                                      flat=flat, debias=debias, replace=replace)
        shim = LayerRng(*KEY)
        mb = rsamplers.build_minibatch(g, np.asarray(tg, dtype=np.int64), params, shim,
                                       batch_id=KEY[2], epoch=KEY[1])
        assert shim.calls == layers, (name, shim.calls)
        store(out, name, mb, params)
        out[f"{name}/graph"] = np.array(gname)
        names.append(name)
    out["cases"] = np.array(names)

    # per-function pins: the first layer's probabilities and the global ones
    for gname in ("g8", "g2"):
        g = graphs[gname]
        prev = np.arange(g.num_nodes, dtype=np.int64)[:: (3 if gname == "g2" else 2)][::-1].copy()
        cand = rsamplers.ladies_candidates(g, prev)
        out[f"probs/{gname}/prev"] = prev
        out[f"probs/{gname}/cand"] = cand
        out[f"probs/{gname}/ladies"] = rsamplers.ladies_probs(g, cand, prev)
        out[f"probs/{gname}/flat"] = rsamplers.flat_probs(g, cand, prev)
        out[f"probs/{gname}/fastgcn"] = rsamplers.fastgcn_probs(g, flat=False)
        out[f"probs/{gname}/fastgcn_flat"] = rsamplers.fastgcn_probs(g, flat=True)
    p = np.array([0.4, 0.1, 0.2, 0.05, 0.25])
    out["debias/probs"] = p
    out["debias/n"] = np.array(9)
    out["debias/coef"] = rsamplers.debias_coefficients(p, 9)

    # GCN arm of the node-wise sampler (the same per-row Philox shim)
    gcn = []
    for name, g, tg, fo in [("gcn_g8", G8, list(range(8)), (2, 2)),
                            ("gcn_g2", G2, t2[:40], (5, 3))]:
        params = mqpipe.SamplerParams(method="gcn", fanout=fo, num_layers=len(fo))
        key = mg.BatchKey(*KEY)
        mb = mqpipe.build_minibatch(g, np.asarray(tg, dtype=np.int64), params, key,
                                    batch_id=KEY[2], epoch=KEY[1])
        out[f"{name}/fanouts"] = np.array(fo)
        out[f"{name}/target_ids"] = mb.target_ids
        out[f"{name}/digest"] = np.frombuffer(bytes.fromhex(mb.digest()), dtype=np.uint8)
        for l, blk in enumerate(mb.layers):
            for k in ("rows", "cols", "values", "src_ids", "dst_ids"):
                out[f"{name}/L{l}/{k}"] = getattr(blk, k)
        gcn.append(name)
    out["gcn_cases"] = np.array(gcn)

    # run_epoch (serial deterministic schedule) with the layer-wise samplers
    # and the GCN arch: the reference's own runtime, its batch rng replaced by
    # the layer stream (a LayerRng per batch) or the node-wise row shim
    rruntime, rnn = mg.rruntime, mg.rnn
    node_rng = rruntime.batch_rng
    Gs = mqpipe.split_masks(G2, ratios=(0.3, 0.1, 0.1), seed=2)
    ep = []
    for name, G, method, extra in (("ladies_1dev", 1, "ladies", dict(nodes_per_layer=96)),
                                   ("ladies_2dev_debias", 2, "ladies",
                                    dict(nodes_per_layer=96, debias=True)),
                                   ("fastgcn_2dev", 2, "fastgcn", dict(nodes_per_layer=128)),
                                   ("gcn_2dev", 2, "gcn", dict(fanout=(4, 3)))):
        if method == "gcn":
            rruntime.batch_rng = node_rng
        else:
            rruntime.batch_rng = lambda config, epoch, bid: LayerRng(config.seed, epoch, bid)
        cfg = rruntime.PipelineConfig(
            num_devices=G, batch_size=64,
            sampler=mqpipe.SamplerParams(method=method, num_layers=2, **extra),
            optimizer="adam", sync_period=1, deterministic=True, seed=5)
        base = rnn.init_model(16, 16, 5, num_layers=2, arch="gcn", seed=5, learning_rate=0.01)
        reps = [base.copy() for _ in range(G)]
        stats, _ = rruntime.run_epoch(Gs, None, reps, cfg, epoch=1)
        k = f"epoch/{name}"
        out[f"{k}/loss_bids"] = np.array(sorted(stats.losses))
        out[f"{k}/losses"] = np.array([stats.losses[b] for b in sorted(stats.losses)])
        out[f"{k}/sync"] = np.array([stats.sync_count, stats.epoch_sync, stats.dropped_targets])
        for l in range(2):
            out[f"{k}/w{l}"] = reps[0].weights[l]
        out[f"{k}/config"] = np.array([G, 64, 5])
        ep.append(name)
    rruntime.batch_rng = node_rng
    out["epoch_cases"] = np.array(ep)
    out["epoch/train_mask"] = Gs.train_mask
    np.savez_compressed(HERE / "layerwise.npz", **out)
    print("wrote", HERE / "layerwise.npz", len(out), "arrays")


if __name__ == "__main__":
    main()
