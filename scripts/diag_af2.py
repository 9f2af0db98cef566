"""Stage-by-stage check of the aggregate-first fused step, window 0, per rep."""
import os
import sys
sys.path.insert(0, "tests")
sys.path.insert(0, ".")
import numpy as np  # noqa
import torch  # noqa
from conftest import load_golden, make_g2  # noqa
import paper_2601_04707_b200 as mq  # noqa
from oracle import nn as onn, sampler as osamp  # noqa
from paper_2601_04707_b200.graph import DeviceGraph  # noqa
from paper_2601_04707_b200.runtime import epoch_permutation  # noqa
from paper_2601_04707_b200._lib import lib  # noqa

lib().mq_set_pdl(int(os.environ.get("PDL", "1")))
gs = load_golden("sampling.npz")
hg = make_g2(gs)
fan, hid, B, seed = (6, 4, 3), 32, 200, 5
mask = gs["g2/mask10"]


def rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-30)


for rep in range(int(os.environ.get("REPS", "3"))):
    g = DeviceGraph.from_csr(hg)
    cache = mq.DeviceCache(g, mask)
    state = mq.init_model(16, hid, 5, num_layers=3, seed=7, learning_rate=0.01)
    model = onn.init_model(16, hid, 5, num_layers=3, seed=7, learning_rate=0.01)
    perm = epoch_permutation(hg.train_mask, seed, 0)
    r = mq.StepRunner(g, state, fanouts=fan, batch_size=B, num_train=perm.size, cache=cache,
                      seed=seed, use_graph=False, pipeline=False, layer0="af")
    r.begin_epoch(0, perm)
    s = r.stream
    sw = r.groups[0].slots[0]
    tw = r.tw
    with torch.cuda.stream(s):
        r._enqueue_prep(sw, s.cuda_stream)
    torch.cuda.synchronize()
    tg = perm[:B]
    mb = osamp.build_minibatch(hg.row_offsets, hg.col_indices, hg.features, hg.labels, tg, fan,
                               seed=seed, epoch=0, batch_id=0, cached_mask=mask)
    logits, cache_o = onn.sage_forward(mb.layers, mb.features, model.weights)
    oloss, _ = onn.batch_loss(logits, mb.target_labels)
    ops = tw.train_ops(state.dev, sw, None, 0, 1)
    out = []
    for name, op in ops:
        with torch.cuda.stream(s):
            op(s.cuda_stream)
        torch.cuda.synchronize()
        if name == "sage_spmm_l0":
            nd = mb.layers[0].num_dst
            agg = onn.block_apply(mb.layers[0], mb.features)
            out.append(("agg0", rel(tw.agg0[:nd, :16].cpu().numpy(), agg)))
        if name == "sage_linear_af_l0":
            nd = mb.layers[0].num_dst
            h1 = np.maximum(cache_o["pre"][0], 0)
            out.append(("act1", rel(tw.act[1][:nd, :hid].cpu().numpy(), h1)))
        if name == "sage_aggregate_l1":
            nd = mb.layers[1].num_dst
            h2 = np.maximum(cache_o["pre"][1], 0)
            out.append(("act2", rel(tw.act[2][:nd, :hid].cpu().numpy(), h2)))
        if name == "sage_head":
            out.append(("loss", abs(float(tw.loss.item()) - oloss) / oloss))
            break
    x0 = sw.x0[:mb.features.shape[0], :16].cpu().numpy()
    out.append(("x0", rel(x0, mb.features)))
    dmb = r.groups[0].minibatch(0, 0)
    for l, (a, b) in enumerate(zip(dmb.layers, mb.layers)):
        ra = a.to_reference()
        for k in ("rows", "cols", "src_ids"):
            ok = ra[k].shape == getattr(b, k).shape and np.array_equal(ra[k], getattr(b, k))
            if not ok:
                out.append((f"L{l}.{k}", float(ra[k].shape[0]) - getattr(b, k).shape[0]))
    out.append(("tg", float(np.array_equal(dmb.target_ids.cpu().numpy(), tg))))
    print(rep, " ".join(f"{k}={v:.2e}" for k, v in out), flush=True)
