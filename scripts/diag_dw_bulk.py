"""Diagnostics: which dW0 entries differ from the oracle when the swapped DW
epilogue uses bulk copies (MQ_TC2_BULK).  Runs the cfg1 fused step eagerly."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
from conftest import make_cfg1  # noqa: E402

import paper_2601_04707_b200 as mq  # noqa: E402
from oracle import nn as onn  # noqa: E402
from oracle import sampler as osamp  # noqa: E402
from paper_2601_04707_b200.graph import DeviceGraph  # noqa: E402
from paper_2601_04707_b200.runtime import epoch_permutation  # noqa: E402

hg = make_cfg1()
rng = np.random.default_rng(0)
mask = np.zeros(hg.num_nodes, bool)
mask[rng.choice(hg.num_nodes, 100, replace=False)] = True
g = DeviceGraph.from_csr(hg)
cache = mq.DeviceCache(g, mask)
fan, B, seed = (10, 5), 1024, 4
for trial in range(int(os.environ.get("TRIALS", "6"))):
    state = mq.init_model(hg.feature_dim, 64, 4, num_layers=2, seed=7, learning_rate=0.01)
    model = onn.init_model(hg.feature_dim, 64, 4, num_layers=2, seed=7, learning_rate=0.01)
    perm = epoch_permutation(hg.train_mask, seed, 0)
    runner = mq.StepRunner(g, state, fanouts=fan, batch_size=B, num_train=perm.size, cache=cache,
                           seed=seed, use_graph=False, pipeline=False, layer0="tf")
    runner.begin_epoch(0, perm)
    if os.environ.get("DEFERRED"):
        runner.tw.grad_src(state.dev)
    s = runner.stream
    sw = runner.groups[0].slots[0]
    with torch.cuda.stream(s):
        runner._enqueue_prep(sw, s.cuda_stream)
        runner._enqueue_train(sw, s.cuda_stream, commit=False)
        runner.tw.materialize_grads(state.dev, s.cuda_stream)
    torch.cuda.synchronize()
    g0 = state.dev.grad(0).cpu().numpy()
    tg = perm[:B]
    mb = osamp.build_minibatch(hg.row_offsets, hg.col_indices, hg.features, hg.labels, tg, fan,
                               seed=seed, epoch=0, batch_id=0, cached_mask=mask)
    logits, c = onn.sage_forward(mb.layers, mb.features, model.weights)
    _, dl = onn.batch_loss(logits, mb.target_labels)
    c["pre"][0] = runner.tw.act[1][:c["pre"][0].shape[0], :c["pre"][0].shape[1]].cpu().numpy()
    r0 = onn.backward(mb.layers, model.weights, c, dl)[0]
    err = np.abs(g0 - r0)
    bad = err > 1e-4 * np.abs(r0).max()
    print(f"trial {trial}: max err {err.max() / np.abs(r0).max():.3e}, bad {bad.sum()} of {bad.size}",
          "rows", np.unique(np.nonzero(bad)[0])[:20], "cols", np.unique(np.nonzero(bad)[1])[:20])
    if bad.any():
        i, j = np.argwhere(bad)[0]
        print("   e.g. got", g0[i, j], "ref", r0[i, j], "ratio", g0[i, j] / r0[i, j])
