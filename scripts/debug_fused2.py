"""Debug: re-run the train half of one window with each GEMM backend on the same
sampled slot and diff every intermediate buffer."""
import sys
import numpy as np
import torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from conftest import load_golden, make_g2
import paper_2601_04707_b200 as mq
from paper_2601_04707_b200._lib import lib
from paper_2601_04707_b200.graph import DeviceGraph
from paper_2601_04707_b200.runtime import epoch_permutation

gs = load_golden("sampling.npz")
hg = make_g2(gs)
mask = gs["g2/mask10"]
fan, H, B, seed = (6, 4, 3), 32, 200, 5
g = DeviceGraph.from_csr(hg)
cache = mq.DeviceCache(g, mask)
state = mq.init_model(hg.feature_dim, H, 5, num_layers=3, seed=7, learning_rate=0.01)
perm = epoch_permutation(hg.train_mask, seed, 0)
r = mq.StepRunner(g, state, fanouts=fan, batch_size=B, num_train=perm.size, cache=cache,
                  seed=seed, use_graph=False, pipeline=False)
r.begin_epoch(0, perm)
s = r.stream
tw = r.tw
for j in range(3):
    with torch.cuda.stream(s):
        r._enqueue_prep(r.slots[0], s.cuda_stream)
    torch.cuda.synchronize()
    snaps = {}
    for backend in (0, 1, 1, 0):
        lib().mq_set_gemm_backend(backend)
        with torch.cuda.stream(s):
            r._enqueue_train(r.slots[0], s.cuda_stream, commit=False)
        torch.cuda.synchronize()
        tw.loss.zero_()
        snap = {"Y0": tw.Y[0], "Y1": tw.Y[1], "act1": tw.act[1], "act2": tw.act[2],
                "dh2": tw.dh[2], "G1": tw.G[1], "dh1": tw.dh[1], "G0": tw.G[0],
                "g": state.dev.flat_g}
        snap = {k: v.detach().cpu().numpy().copy() for k, v in snap.items()}
        if backend in snaps:
            same = {k: bool(np.array_equal(snaps[backend][k], snap[k])) for k in snap}
            print(f"window {j} backend {backend} rerun bit-identical: {same}")
        snaps[backend] = snap
    c = r.read_counts(0)
    print("counts", c)
    for k in snaps[0]:
        a, b = snaps[0][k], snaps[1][k]
        err = np.abs(a - b).max() / max(np.abs(a).max(), 1e-30)
        print(f"window {j} {k:5s} ffma-vs-tc rel {err:.2e}")
