"""Phase timeline of CTA 0 of the fused head and the tcgen05 GEMMs on the
Reddit-shaped step (MQ_TC_TRACE library: libmqgnn_trace.so)."""
import ctypes as C
import os
import sys
os.environ["MQGNN_LIB"] = os.environ.get("MQ_TRACE_LIB") or os.path.join(os.path.dirname(__file__), "..", "paper_2601_04707_b200",
                                       "libmqgnn_trace.so")
import torch
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import bench  # noqa: E402
import paper_2601_04707_b200 as mq  # noqa: E402
from paper_2601_04707_b200._lib import lib  # noqa: E402
from paper_2601_04707_b200.runtime import epoch_permutation  # noqa: E402

sys.argv = [sys.argv[0]] + sys.argv[1:]
args = bench.parse()
dev = torch.device("cuda", 0)
sg, fanouts, _ = bench.build_inputs(args, "cuda:0")
g = mq.DeviceGraph.from_csr(sg, device=dev)
cache = mq.refresh_cache(g, mq.cache_probs_degree(g), args.cache_fraction, mq.RefreshStream(0, 0))
model = mq.init_model(g.feature_dim, args.hidden, g.num_classes, num_layers=len(fanouts), seed=0,
                      learning_rate=1e-3, device=dev)
n_train = int(g.train_mask.sum())
runner = mq.StepRunner(g, model, fanouts=fanouts, batch_size=1024, num_train=n_train, cache=cache,
                       layer0=args.layer0)
runner.capture()
runner.begin_epoch(0, epoch_permutation(g.train_mask, 0, 0))
runner.steps(8)
torch.cuda.synchronize()
gi, q = runner._last
sw = runner.groups[gi].slots[q]
ops = dict(runner.tw.train_ops(runner.dm, sw))
buf = (C.c_ulonglong * 16)()
for rep in range(3):
    with torch.cuda.stream(runner.stream):
        ops["sage_head"](runner.stream.cuda_stream)
    torch.cuda.synchronize()
lib().dll.mq_debug_head_trace(buf)
t = [int(x) for x in buf]
print("head phases (us from entry):", " ".join(f"{i}:{(t[i] - t[0]) / 1e3:.2f}" for i in range(8)))
print("  1 W/W^T staged, 2 aggregated, 3 logits, 4 CE, 5 dt atomics, 6 dW partial, 7 end")
cta = (C.c_ulonglong * (256 * 8))()
lib().dll.mq_debug_head_cta(cta)
n_cta = -(-1024 // int(os.environ.get("MQ_HEAD_ROWS_TRACE", "4")))
rows = [[int(cta[8 * b + i]) for i in range(8)] for b in range(n_cta)]
t0 = min(r[0] for r in rows)
import statistics as _st
print("  per-CTA phase durations (us) min / median / max over", n_cta, "CTAs; start skew",
      f"{(max(r[0] for r in rows) - t0) / 1e3:.2f}, last end {(max(r[7] for r in rows) - t0) / 1e3:.2f}")
for i in range(1, 8):
    d = [(r[i] - r[i - 1]) / 1e3 for r in rows]
    print(f"    phase {i}: {min(d):6.2f} {_st.median(d):6.2f} {max(d):6.2f}")

# ---- in-step timeline of one window: first CTA entry / last CTA exit per kernel
names = {0: "tc FWD", 1: "tc DW", 2: "tc FCAT", 3: "tc DCAT", 4: "tc DX", 5: "aggregate",
         6: "head", 7: "scatter", 8: "adam"}
tl = (C.c_ulonglong * 64)()
for tag in ("fused", "train", "tc"):
    getattr(lib().dll, f"mq_debug_timeline_{tag}")(tl, 1)
for rep in range(2):
    torch.cuda.synchronize()
    for tag in ("fused", "train", "tc"):
        getattr(lib().dll, f"mq_debug_timeline_{tag}")(tl, 1)
    runner.steps(1)  # one window graph (prep forked only at group boundaries)
    torch.cuda.synchronize()
rows = {}
for tag in ("fused", "train", "tc"):
    getattr(lib().dll, f"mq_debug_timeline_{tag}")(tl, 0)
    for i in range(32):
        a, b = int(tl[2 * i]), int(tl[2 * i + 1])
        if a != 2 ** 64 - 1 and b:
            rows[i] = (a, b)
t0 = min(a for a, _ in rows.values())
prev = None
for i, (a, b) in sorted(rows.items(), key=lambda kv: kv[1][0]):
    gap = "" if prev is None else f" gap {(a - prev) / 1e3:5.2f}"
    print(f"  {names.get(i, i):10s} {(a - t0) / 1e3:7.2f} -> {(b - t0) / 1e3:7.2f} us "
          f"({(b - a) / 1e3:5.2f}){gap}")
    prev = b

# ---- the in-step head's per-CTA phases (the last head launch was in-step)
lib().dll.mq_debug_head_cta(cta)
rows = [[int(cta[8 * b + i]) for i in range(8)] for b in range(n_cta)]
t0 = min(r[0] for r in rows)
print("  in-step head, per-CTA phase durations (us) min / median / max; start skew",
      f"{(max(r[0] for r in rows) - t0) / 1e3:.2f}, last end {(max(r[7] for r in rows) - t0) / 1e3:.2f}")
for i in range(1, 8):
    d = [(r[i] - r[i - 1]) / 1e3 for r in rows]
    print(f"    phase {i}: {min(d):6.2f} {_st.median(d):6.2f} {max(d):6.2f}")
