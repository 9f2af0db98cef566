"""Layer-wise samplers on the Reddit-shaped graph: device
batch build (build_minibatch: LADIES / FastGCN / GCN node-wise) and the
per-op GCN training step (loss_and_grads + adam_step), seeds/s, against the
CPU oracle restatement on the same batches (and a bit-exact check of the
first batch's blocks against it).

    python scripts/bench_layerwise.py [--shape reddit] [--batches 20]

Prints one JSON line per method.  The device path synchronises per layer
(the reference API returns arrays), so these are API-path numbers.
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import paper_2601_04707_b200 as mq  # noqa: E402
from paper_2601_04707_b200 import synth  # noqa: E402
from paper_2601_04707_b200._lib import lib  # noqa: E402
from oracle import layerwise as olw  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", default="reddit")
    ap.add_argument("--batches", type=int, default=20)
    ap.add_argument("--budget", type=int, default=512)
    ap.add_argument("--cpu-batches", type=int, default=2)
    ap.add_argument("--methods", default="ladies,fastgcn,gcn")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    sg, fanouts = synth.generate_shape(args.shape, seed=0, device="cuda:0")
    g = mq.DeviceGraph.from_csr(sg, device=dev)
    ro = sg.row_offsets.cpu().numpy().astype(np.int64)
    col = sg.col_indices.cpu().numpy().astype(np.int64)
    train = np.flatnonzero(g.train_mask)
    rng = np.random.default_rng(0)
    batches = [rng.choice(train, 1024, replace=False) for _ in range(args.batches + 2)]
    L = len(fanouts)
    for method in args.methods.split(","):
        if method == "gcn":
            params = mq.SamplerParams(method="gcn", fanout=tuple(fanouts), num_layers=L)
        else:
            params = mq.SamplerParams(method=method, nodes_per_layer=args.budget, num_layers=L)
        state = mq.init_model(g.feature_dim, 64, g.num_classes, num_layers=L, arch="gcn", seed=0,
                              device=dev)
        t_fg = None
        if method == "fastgcn":  # per-graph global probabilities (cached), timed once
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            mq.fastgcn_probs(g)
            torch.cuda.synchronize()
            t_fg = time.perf_counter() - t0
        for b in range(2):  # warm-up
            mb = mq.build_minibatch(g, batches[b], params, mq.PhiloxStream(0, 0, b), batch_id=b)
            loss, grads, _ = mq.loss_and_grads(mb, state)
            mq.adam_step(state, grads)
        lib().mq_prof_enable(1)
        lib().mq_prof_reset()
        torch.cuda.synchronize()
        t_build = t_step = 0.0
        nnz = n_in = 0
        for b in range(2, args.batches + 2):
            t0 = time.perf_counter()
            mb = mq.build_minibatch(g, batches[b], params, mq.PhiloxStream(0, 0, b), batch_id=b)
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            loss, grads, _ = mq.loss_and_grads(mb, state)
            mq.adam_step(state, grads)
            torch.cuda.synchronize()
            t2 = time.perf_counter()
            t_build += t1 - t0
            t_step += t2 - t1
            nnz += sum(blk.nnz for blk in mb.layers)
            n_in += int(mb.input_ids.numel())
        nb = args.batches
        prof = read_prof()
        lib().mq_prof_enable(0)
        # CPU oracle on the first timed batches (same draws)
        cpu_s, exact = 0.0, None
        dh = olw.a_hat_degrees(ro, col)
        for b in range(2, 2 + args.cpu_batches):
            r = olw.LayerRng(0, 0, b)
            t0 = time.perf_counter()
            if method == "ladies":
                blocks, _ = olw.sample_ladies(ro, col, batches[b], args.budget, L, r, deg_hat=dh)
            elif method == "fastgcn" and col.size < 20_000_000:
                blocks = olw.sample_fastgcn(ro, col, batches[b], args.budget, L, r, deg_hat=dh,
                                            probs=fg_probs(ro, col, dh))
            else:
                blocks = None
            cpu_s += time.perf_counter() - t0
            if blocks is not None and b == 2:
                mb = mq.build_minibatch(g, batches[b], params, mq.PhiloxStream(0, 0, b), batch_id=b)
                exact = all(
                    np.array_equal(blk.to_reference()[k], getattr(ob, k))
                    for blk, ob in zip(mb.layers, blocks)
                    for k in ("rows", "cols", "values", "effective_values", "src_ids"))
        line = {"metric": f"{method} batch build + GCN step (per-op API)", "shape": args.shape,
                "method": method, "budget": args.budget if method != "gcn" else None,
                "fanouts": list(fanouts) if method == "gcn" else None, "batches": nb,
                "build_ms": 1e3 * t_build / nb, "step_ms": 1e3 * t_step / nb,
                "seeds_per_s": 1024 * nb / (t_build + t_step),
                "build_seeds_per_s": 1024 * nb / t_build,
                "mean_nnz": nnz / nb, "mean_input_rows": n_in / nb,
                "fastgcn_probs_s": t_fg,
                "cpu_oracle_build_ms": (1e3 * cpu_s / args.cpu_batches) if method != "gcn" else None,
                "bit_exact_vs_oracle_first_batch": exact,
                "device_ms_per_batch": {k: v / nb for k, v in prof.items()}}
        print(json.dumps(line), flush=True)


_FG = {}


def read_prof():
    import ctypes as C
    n = lib().mq_prof_num_kernels()
    ms = (C.c_double * n)()
    cnt = (C.c_int64 * n)()
    lib().mq_prof_read(ms, cnt, n)
    return {lib().mq_prof_kernel_name(i).decode(): ms[i] for i in range(n) if cnt[i]}


def fg_probs(ro, col, dh):
    if "p" not in _FG:
        _FG["p"] = olw.fastgcn_probs(ro, col, dh)
    return _FG["p"]


if __name__ == "__main__":
    main()
