"""Time the fused head kernel variants on the Reddit-shaped workload (GPU)."""
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
import bench
import paper_2601_04707_b200 as mq
from paper_2601_04707_b200._lib import lib, ptr
from paper_2601_04707_b200.profiling import _time
from paper_2601_04707_b200.runtime import epoch_permutation

args = bench.parse()
dev = torch.device("cuda", 0)
sg, fanouts, _ = bench.build_inputs(args, "cuda:0")
g = mq.DeviceGraph.from_csr(sg, device=dev)
cache = mq.refresh_cache(g, mq.cache_probs_degree(g), args.cache_fraction, mq.RefreshStream(args.seed, 0))
model = mq.init_model(g.feature_dim, args.hidden, g.num_classes, num_layers=len(fanouts), seed=0,
                      learning_rate=1e-3, device=dev)
n_train = int(g.train_mask.sum())
runner = mq.StepRunner(g, model, fanouts=fanouts, batch_size=1024, num_train=n_train, cache=cache)
runner.capture()
runner.begin_epoch(0, epoch_permutation(g.train_mask, 0, 0))
runner.steps(8)
torch.cuda.synchronize()
tw, dm = runner.tw, runner.dm
gi, q = runner._last
sw = runner.groups[gi].slots[q]
L = tw.L
d, ld = tw.dims, tw.ld_in
hb0 = sw.hops[0]
lb = lib()


def head(dh):
    return lambda s: lb.mq_sage_head(ptr(hb0.row_ptr), ptr(hb0.cols), ptr(hb0.vals),
                                     ptr(sw.n_targets), sw.batch_size, ptr(tw.h_in(L - 1, sw)),
                                     ld[L - 1], d[L - 1], ptr(model.weights[L - 1]), tw.C,
                                     ptr(sw.labels), None, ptr(dh), ld[L - 1], ptr(tw.loss),
                                     ptr(sw.key), 1, None, 0, ptr(dm.nonfinite),
                                     ptr(tw.head_scratch), s)


print("head full     %.2f us" % _time(head(tw.dh[L - 1]), runner.stream, 20, 3))
print("head no dh    %.2f us" % _time(head(None), runner.stream, 20, 3))
# degree skew of the hop-0 block's columns (atomic contention on dh rows)
c = runner.read_counts()
nnz = c["hops"][0][2]
cols = hb0.cols[:nnz].cpu().numpy()
cnt = np.bincount(cols)
print("hop0 nnz", nnz, "distinct cols", (cnt > 0).sum(), "max per col", cnt.max(),
      "top10", np.sort(cnt)[-10:])
c1 = sw.hops[1].cols[:c["hops"][1][2]].cpu().numpy()
cnt1 = np.bincount(c1)
print("hop1 distinct cols", (cnt1 > 0).sum(), "max per col", cnt1.max())
