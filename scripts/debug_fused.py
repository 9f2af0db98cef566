"""Debug: per-window gradient error of the fused step vs the oracle, per GEMM backend."""
import sys
import numpy as np
import torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from conftest import load_golden, make_g2
import paper_2601_04707_b200 as mq
from oracle import nn as onn, sampler as osamp
from paper_2601_04707_b200._lib import lib
from paper_2601_04707_b200.graph import DeviceGraph
from paper_2601_04707_b200.runtime import epoch_permutation

gs = load_golden("sampling.npz")
hg = make_g2(gs)
mask = gs["g2/mask10"]
fan, H, B, seed = (6, 4, 3), 32, 200, 5
for backend in (0, 1):
    lib().mq_set_gemm_backend(backend)
    g = DeviceGraph.from_csr(hg)
    cache = mq.DeviceCache(g, mask)
    state = mq.init_model(hg.feature_dim, H, 5, num_layers=3, seed=7, learning_rate=0.01)
    model = onn.init_model(hg.feature_dim, H, 5, num_layers=3, seed=7, learning_rate=0.01)
    perm = epoch_permutation(hg.train_mask, seed, 0)
    r = mq.StepRunner(g, state, fanouts=fan, batch_size=B, num_train=perm.size, cache=cache,
                      seed=seed, use_graph=False, pipeline=False)
    r.begin_epoch(0, perm)
    s = r.stream
    for j in range(4):
        with torch.cuda.stream(s):
            r._enqueue_prep(r.slots[0], s.cuda_stream)
            r._enqueue_train(r.slots[0], s.cuda_stream, commit=False)
        torch.cuda.synchronize()
        c = r.read_counts(0)
        r.tw.loss.zero_()
        grads = [state.dev.grad(l).cpu().numpy() for l in range(3)]
        tg = perm[j * B:(j + 1) * B]
        mb = osamp.build_minibatch(hg.row_offsets, hg.col_indices, hg.features, hg.labels, tg, fan,
                                   seed=seed, epoch=0, batch_id=j, cached_mask=mask)
        _, og, _ = onn.loss_and_grads(mb.layers, mb.features, mb.target_labels, model.weights)
        errs = [float(np.abs(a - b).max() / np.abs(b).max()) for a, b in zip(grads, og)]
        print(f"backend {backend} window {j} counts {c['hops']} errs {['%.2e' % e for e in errs]}")
        if backend == 1 and errs[0] > 1e-4:
            d = np.abs(grads[0] - og[0])
            rows = np.where(d.max(axis=1) > 1e-4 * np.abs(og[0]).max())[0]
            cols = np.where(d.max(axis=0) > 1e-4 * np.abs(og[0]).max())[0]
            print("  bad dW0 rows", rows[:40], "cols", cols[:70])
