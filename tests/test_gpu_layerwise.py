"""GPU parity of the layer-wise samplers (LADIES / FastGCN, flat / debias /
with replacement) and the GCN node-wise arm against the reference-made
fixtures (tests/golden/make_golden_layerwise.py): blocks, f64 values,
effective values, sample probabilities, src ids and the batch digest are
compared bit-exactly; the GCN arch's forward/backward against the oracle at
fp32 tolerance."""

import numpy as np
import pytest
import torch

from conftest import GOLDEN, HostGraph, load_golden, make_g2, make_g8
from oracle import layerwise as olw
from oracle import sampler as osamp

pytestmark = pytest.mark.gpu

LW = np.load(GOLDEN / "layerwise.npz")


@pytest.fixture(scope="module")
def graphs():
    import paper_2601_04707_b200 as mq
    samp = load_golden("sampling.npz")
    g2 = make_g2(samp)
    assert np.array_equal(g2.row_offsets, LW["graph/g2/row_offsets"])
    feats9 = np.random.default_rng(42).standard_normal((9, 3)).astype(np.float32)
    g9 = HostGraph(LW["graph/g9/row_offsets"], LW["graph/g9/col_indices"], feats9,
                   np.array([0, 1, 0, 1, 0, 1, 0, 1, 0], np.int32), 2)
    dev = torch.device("cuda", 0)
    return {name: mq.DeviceGraph.from_csr(h, device=dev)
            for name, h in (("g8", make_g8()), ("g9", g9), ("g2", g2))}


def _params(case):
    import paper_2601_04707_b200 as mq
    budget, layers, flat, debias, replace = LW[f"{case}/params"].tolist()
    return mq.SamplerParams(method=str(LW[f"{case}/method"]), nodes_per_layer=budget,
                            num_layers=layers, flat=bool(flat), debias=bool(debias),
                            replace=bool(replace))


@pytest.mark.parametrize("case", [str(c) for c in LW["cases"]])
def test_layerwise_minibatch_bit_exact(graphs, case):
    import paper_2601_04707_b200 as mq
    g = graphs[str(LW[f"{case}/graph"])]
    seed, epoch, batch = LW[f"{case}/key"].tolist()
    req = np.array([8, 1, 8, 6]) if case == "g9_ladies_drop" else LW[f"{case}/target_ids"]
    mb = mq.build_minibatch(g, req, _params(case), mq.PhiloxStream(seed, epoch, batch),
                            batch_id=batch, epoch=epoch)
    assert mb.dropped_targets == int(LW[f"{case}/dropped"])
    np.testing.assert_array_equal(mb.target_ids.cpu().numpy(), LW[f"{case}/target_ids"])
    np.testing.assert_array_equal(mb.target_labels.cpu().numpy(), LW[f"{case}/labels"])
    for l, blk in enumerate(mb.layers):
        ref = blk.to_reference()
        for k in ("rows", "cols", "values", "effective_values", "src_ids", "dst_ids",
                  "sample_probs"):
            np.testing.assert_array_equal(ref[k], LW[f"{case}/L{l}/{k}"], err_msg=f"{case} L{l} {k}")
        # the forward's f32 weights are the effective values cast (nn.py:86)
        np.testing.assert_array_equal(blk.values.cpu().numpy(),
                                      LW[f"{case}/L{l}/effective_values"].astype(np.float32))
        rp = blk.row_ptr.cpu().numpy()
        assert rp[0] == 0 and rp[-1] == blk.nnz
        np.testing.assert_array_equal(np.repeat(np.arange(blk.num_dst), np.diff(rp)), ref["rows"])
    np.testing.assert_array_equal(mb.features.cpu().numpy()[:, :LW[f"{case}/features"].shape[1]],
                                  LW[f"{case}/features"])
    assert bytes.fromhex(mb.digest()) == LW[f"{case}/digest"].tobytes()


@pytest.mark.parametrize("g", ["g8", "g2"])
def test_fastgcn_probs_bit_exact(graphs, g):
    import paper_2601_04707_b200 as mq
    for flat, key in ((False, "fastgcn"), (True, "fastgcn_flat")):
        got = mq.fastgcn_probs(graphs[g], flat=flat).cpu().numpy()
        np.testing.assert_array_equal(got, LW[f"probs/{g}/{key}"])


@pytest.mark.parametrize("case", [str(c) for c in LW["gcn_cases"]])
def test_gcn_node_wise_arm_bit_exact(graphs, case):
    import paper_2601_04707_b200 as mq
    g = graphs[case.split("_")[1]]
    fo = tuple(LW[f"{case}/fanouts"].tolist())
    params = mq.SamplerParams(method="gcn", fanout=fo, num_layers=len(fo))
    mb = mq.build_minibatch(g, LW[f"{case}/target_ids"], params, mq.PhiloxStream(5, 2, 9),
                            batch_id=9, epoch=2)
    for l, blk in enumerate(mb.layers):
        ref = blk.to_reference()
        for k in ("rows", "cols", "values", "src_ids", "dst_ids"):
            np.testing.assert_array_equal(ref[k], LW[f"{case}/L{l}/{k}"], err_msg=f"{case} L{l} {k}")
    assert bytes.fromhex(mb.digest()) == LW[f"{case}/digest"].tobytes()


def test_layer_uniforms_host_match_oracle():
    import ctypes as C

    from paper_2601_04707_b200._lib import lib
    out = (C.c_double * 64)()
    lib().mq_layer_uniforms_host(7, 3, 11, 2, 64, out)
    np.testing.assert_array_equal(np.frombuffer(out, dtype=np.float64),
                                  olw.layer_uniforms(7, 3, 11, 2, 64))


def _oracle_gcn(blocks, feats, labels, weights):
    """GCN forward / loss / backward in NumPy (nn.py:102-113, 141-180 gcn arm)."""
    h = feats.astype(np.float32)
    ins, pre = [], []
    for l, b in enumerate(blocks):
        agg = np.zeros((b["n_dst"], h.shape[1]), np.float32)
        np.add.at(agg, b["rows"], b["eff"].astype(np.float32)[:, None] * h[b["cols"]])
        z = agg @ weights[l]
        ins.append((h, agg))
        pre.append(z)
        h = np.maximum(z, 0) if l < len(blocks) - 1 else z
    sh = h - h.max(1, keepdims=True)
    ex = np.exp(sh)
    den = ex.sum(1, keepdims=True)
    loss = -(sh - np.log(den))[np.arange(len(labels)), labels].sum()
    dz = ex / den
    dz[np.arange(len(labels)), labels] -= 1
    grads = [None] * len(blocks)
    for l in range(len(blocks) - 1, -1, -1):
        hin, agg = ins[l]
        if l < len(blocks) - 1:
            dz = dz * (pre[l] > 0)
        grads[l] = agg.T @ dz
        if l > 0:
            dt = dz @ weights[l].T
            dh = np.zeros((hin.shape[0], dt.shape[1]), np.float32)
            np.add.at(dh, blocks[l]["cols"], blocks[l]["eff"].astype(np.float32)[:, None]
                      * dt[blocks[l]["rows"]])
            dz = dh
    return float(loss), h, grads


@pytest.mark.parametrize("method", ["ladies", "fastgcn", "gcn"])
def test_gcn_arch_forward_backward(graphs, method):
    import paper_2601_04707_b200 as mq
    g = graphs["g2"]
    samp = load_golden("sampling.npz")
    feats, labels = samp["g2/features"], samp["g2/labels"]
    tg = np.random.default_rng(5).choice(2000, 128, replace=False)
    if method == "gcn":
        params = mq.SamplerParams(method="gcn", fanout=(5, 3), num_layers=2)
    else:
        params = mq.SamplerParams(method=method, nodes_per_layer=256, num_layers=2)
    mb = mq.build_minibatch(g, tg, params, mq.PhiloxStream(1, 0, 3), batch_id=3)
    state = mq.init_model(16, 32, 5, num_layers=2, arch="gcn", seed=4)
    loss, grads, logits = mq.loss_and_grads(mb, state)
    blocks = []
    for blk in mb.layers:
        r = blk.to_reference()
        blocks.append(dict(rows=r["rows"], cols=r["cols"], eff=r["effective_values"],
                           n_dst=blk.num_dst))
    ws = [w.cpu().numpy() for w in state.weights]
    kept = mb.target_ids.cpu().numpy()
    rl, rlog, rg = _oracle_gcn(blocks, feats[mb.input_ids.cpu().numpy()], labels[kept], ws)
    assert abs(loss - rl) <= 1e-5 * abs(rl)
    lg = logits.cpu().numpy()
    assert np.abs(lg - rlog).max() <= 1e-5 * np.abs(rlog).max()
    for a, b in zip(grads, rg):
        a = a.cpu().numpy()
        assert np.abs(a - b).max() <= 2e-5 * np.abs(b).max()
    mq.adam_step(state, grads)


def test_layerwise_errors(graphs):
    import paper_2601_04707_b200 as mq
    g = graphs["g9"]
    with pytest.raises(mq.SamplingError):
        mq.sample_ladies(g, [8, 8], 3, 1, mq.PhiloxStream(0, 0, 0))
    with pytest.raises(mq.SamplingError):
        mq.sample_fastgcn(g, [], 3, 1, mq.PhiloxStream(0, 0, 0))


@pytest.mark.parametrize("case", [str(c) for c in LW["epoch_cases"]])
def test_run_epoch_layerwise_and_gcn_match_reference(case):
    """run_epoch with LADIES / FastGCN / the GCN node-wise arm and the GCN
    arch (the per-op serial schedule) against the reference's own run_epoch:
    per-batch losses and the final weights."""
    import paper_2601_04707_b200 as mq
    samp = load_golden("sampling.npz")
    hg = make_g2(samp)
    hg.train_mask = LW["epoch/train_mask"]
    g = mq.DeviceGraph.from_csr(hg, device=torch.device("cuda", 0))
    G, B, seed = LW[f"epoch/{case}/config"].tolist()
    method = case.split("_")[0]
    if method == "gcn":
        params = mq.SamplerParams(method="gcn", fanout=(4, 3), num_layers=2)
    else:
        params = mq.SamplerParams(method=method, nodes_per_layer=128 if method == "fastgcn" else 96,
                                  num_layers=2, debias="debias" in case)
    cfg = mq.PipelineConfig(num_devices=G, batch_size=B, sampler=params, optimizer="adam",
                            sync_period=1, deterministic=True, seed=seed)
    base = mq.init_model(16, 16, 5, num_layers=2, arch="gcn", seed=5, learning_rate=0.01)
    reps = [base.copy() for _ in range(G)]
    stats, _ = mq.run_epoch(g, None, reps, cfg, epoch=1)
    bids = LW[f"epoch/{case}/loss_bids"]
    assert sorted(stats.losses) == bids.tolist()
    got = np.array([stats.losses[b] for b in bids])
    ref = LW[f"epoch/{case}/losses"]
    np.testing.assert_allclose(got, ref, rtol=1e-4)
    assert [stats.sync_count, stats.epoch_sync, stats.dropped_targets] == \
        LW[f"epoch/{case}/sync"].tolist()
    for l in range(2):
        w = reps[0].weights[l].cpu().numpy()
        ref_w = LW[f"epoch/{case}/w{l}"]
        assert np.abs(w - ref_w).max() <= 1e-4 * np.abs(ref_w).max()
        for r in reps[1:]:  # replicas identical after the epoch barrier
            np.testing.assert_array_equal(r.weights[l].cpu().numpy(), w)
