"""Per-phase timeline of CTA 0 of the tcgen05 GEMMs (needs the MQ_TC_TRACE build:
MQ_BUILD_OUT=paper_2601_04707_b200/libmqgnn_trace.so MQ_BUILD_TAG=_trace
MQ_EXTRA_NVCC_FLAGS=-DMQ_TC_TRACE python -m paper_2601_04707_b200._build)."""
import ctypes as C
import os
import sys
os.environ["MQGNN_LIB"] = os.path.join(os.path.dirname(__file__), "..", "paper_2601_04707_b200",
                                       "libmqgnn_trace.so")
import numpy as np
import torch
sys.path.insert(0, '.')
import bench
import paper_2601_04707_b200 as mq
from paper_2601_04707_b200._lib import lib
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
gi, q = runner._last
sw = runner.groups[gi].slots[q]
ops = dict(runner.tw.train_ops(runner.dm, sw))
buf = (C.c_ulonglong * 32)()
for name in ("sage_transform_l0", "sage_transform_bwd_l0"):
    for rep in range(3):
        with torch.cuda.stream(runner.stream):
            ops[name](runner.stream.cuda_stream)
        torch.cuda.synchronize()
    lib().dll.mq_debug_tc_trace(buf)
    t = np.array(list(buf), dtype=np.int64)
    base = t[0]
    rel = {i: (t[i] - base) / 1e3 for i in range(32) if t[i] >= base and t[i] - base < 1e9}
    print(name, " ".join(f"{i}:{v:.2f}" for i, v in sorted(rel.items())))
print("counts", runner.read_counts())
