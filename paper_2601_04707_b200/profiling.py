"""Per-launch device timing of the step's kernels (bench / roofline evidence).

Each op of the fused step (FusedTrainWorkspace.train_ops, the optimizer and
the prep stages of mq_prep_batches selected by stage_mask) is captured
``reps`` times back to back into one CUDA graph on the runner's train stream
and the graph is replayed under CUDA events: the average is that kernel's
warm, in-graph launch duration — the same inputs, buffers and L2 state as in
the step, without per-launch event or host overhead.  Mutable state touched
by the ops (weights, moments, counters, loss) is snapshotted and restored.

Algorithmic bytes / flops per launch follow SURVEY.md §8(d) and DESIGN.md §3.
"""

from __future__ import annotations

import torch

from ._lib import lib
from .engine import capture_graph
from .prep import PREP_GATHER, PREP_LABELS, PREP_RELABEL, PREP_SAMPLE


def _time(fn, stream, reps: int, iters: int) -> float:
    g = torch.cuda.CUDAGraph()
    with capture_graph(g, stream):
        for _ in range(reps):
            fn(torch.cuda.current_stream().cuda_stream)
    with torch.cuda.stream(stream):
        g.replay()  # warm
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(iters):
            g.replay()
        e1.record(stream)
    e1.synchronize()
    return e0.elapsed_time(e1) * 1e3 / (reps * iters)  # us per launch


def op_models(counts: dict, dims: list, fanouts, Q: int, cached: bool, n_params: int,
              num_classes: int, feature_dim: int) -> dict:
    """name -> {"bytes": algorithmic bytes per launch, "flops": fp32 GEMM flops,
    "units": what one launch covers}."""
    hops = counts["hops"]
    L = len(fanouts)
    B = counts["n_targets"]
    C = num_classes
    m = {}
    samp = relab = samp_sec = relab_sec = 0.0
    for h, (nd, ns, nnz) in enumerate(hops):
        samp += nd * (4 + 16 + (16 if cached else 0) + 4) + nnz * (4 + 4 + (8 if cached else 0))
        relab += 4 * (nnz + nd) + 4 * (nnz + ns) + 4 * (nd + 1)
        # the same work counted in the 32-byte sectors a random access moves:
        # sampler = offsets (+ hot offsets) per row and one column sector per
        # pick (+ its hot-arc entry); relabel = one node-word sector per
        # first-slot atomic, flag read and column read per pick, per label
        # store, per hop-0 mark and per restore (last hop)
        samp_sec += 32 * (nd * (2 if cached else 1) + nnz * (2 if cached else 1))
        relab_sec += 32 * (3 * nnz + (ns - nd) + (nd if h == 0 else 0)
                           + (ns if h == L - 1 else 0))
    n_in = hops[-1][1]
    m["prep_sample"] = {"bytes": Q * samp, "sector_bytes": Q * (samp + samp_sec),
                        "units": f"{Q} batches x {L} hops"}
    m["prep_relabel"] = {"bytes": Q * relab, "sector_bytes": Q * (relab + relab_sec),
                         "units": f"{Q} batches x {L} hops"}
    m["prep_gather"] = {"bytes": Q * (2 * 4 * feature_dim * n_in + 8 * n_in),
                        "units": f"{Q} batches"}
    m["prep_pass"] = {"bytes": m["prep_sample"]["bytes"] + m["prep_relabel"]["bytes"]
                      + m["prep_gather"]["bytes"] + Q * 12 * B,
                      "units": f"{Q} batches (sample + relabel + gather + labels)"}
    for l in range(L - 1):
        nd, ns, nnz = hops[L - 1 - l]
        d, dout = dims[l], dims[l + 1]
        fl = 2.0 * ns * d * 2 * dout
        m[f"sage_transform_l{l}"] = {"bytes": 4 * (ns * d + 2 * d * dout + ns * 2 * dout),
                                     "flops": fl, "units": "1 batch"}
        # compulsory: each Y row read once, act written, triplets read
        m[f"sage_aggregate_l{l}"] = {"bytes": 4 * ns * 2 * dout + 4 * nd * dout + 8 * nnz
                                     + 4 * (nd + 1), "units": "1 batch"}
        m[f"sage_scatter_bwd_l{l}"] = {"bytes": 2 * 4 * nd * dout + 4 * ns * 2 * dout + 8 * nnz,
                                       "units": "1 batch"}
        # dW = h^T G (+ for l > 0 the input gradient dh = G W^T: one more read
        # of G and W, one write of dh)
        m[f"sage_transform_bwd_l{l}"] = {
            "bytes": 4 * (ns * d + ns * 2 * dout + 2 * d * dout)
            + (4 * (ns * 2 * dout + 2 * d * dout + ns * d) if l > 0 else 0),
            "flops": fl * (2 if l > 0 else 1), "units": "1 batch"}
        if l == 0:  # aggregate-first input layer (mq_spmm_fwd + mq_sage_linear_af[_bwd])
            m["sage_spmm_l0"] = {"bytes": 4 * d * (nnz + nd) + 8 * nnz + 4 * (nd + 1),
                                 "units": "1 batch"}
            m["sage_linear_af_l0"] = {"bytes": 4 * (nd * 2 * d + 2 * d * dout + nd * dout),
                                      "flops": 2.0 * nd * 2 * d * dout, "units": "1 batch"}
            m["sage_linear_af_bwd_l0"] = {"bytes": 4 * (nd * 2 * d + 2 * nd * dout),
                                          "flops": 2.0 * nd * 2 * d * dout, "units": "1 batch"}
    nd, ns, nnz = hops[0]
    d = dims[L - 1]
    m["sage_head"] = {"bytes": 4 * d * ns + 8 * nnz + 4 * 2 * d * C + 4 * B
                      + 4 * d * (nnz + nd), "flops": 3 * 2.0 * nd * 2 * d * C,
                      "units": "1 batch"}
    m["optimizer"] = {"bytes": 4 * n_params * 7, "units": f"{n_params} parameters"}
    return m


def op_table(runner, reps: int = 20, iters: int = 3) -> dict:
    """Time every op of the runner's fused step on its last trained slot."""
    if not runner.fused:
        raise ValueError("op_table profiles the fused step")
    torch.cuda.synchronize(runner.device)
    dm = runner.dm
    gi, q = runner._last
    grp = runner.groups[gi]
    sw = grp.slots[q]
    counts = runner.read_counts()
    state = [dm.flat_w, dm.flat_m, dm.flat_v, dm.step_dev, dm.flat_g, dm.nonfinite,
             runner.tw.loss, runner.cursor]
    if runner.cache is not None:
        state.append(runner.cache.hit_miss)
    snap = [t.clone() for t in state]
    ops = list(runner.tw.train_ops(dm, sw, ring=None, ring_len=0, world=runner.world))
    ops.append(("optimizer", lambda s: runner.tw.launch_optimizer(dm, runner.optimizer, s)))
    host = runner._prep_desc(gi, True)  # host-staged descriptor: no batch plan
    # prep_relabel alone re-runs the marks / first slots that the full pass
    # folds into the sampler; prep_pass is the whole batched pass as the step runs it
    for name, mask in (("prep_sample", PREP_SAMPLE), ("prep_relabel", PREP_RELABEL),
                       ("prep_gather", PREP_GATHER),
                       ("prep_pass", PREP_SAMPLE | PREP_RELABEL | PREP_GATHER | PREP_LABELS)):
        def prep_op(s, mask=mask):
            host.stage_mask = mask
            try:
                grp.launch(host, s)
            finally:
                host.stage_mask = 0
        ops.append((name, prep_op))
    out = {}
    # each op's replays run without programmatic dependent launch: otherwise
    # copy k+1 of the same op launches into copy k's SMs and inflates both
    pdl = int(lib().mq_get_pdl())
    lib().mq_set_pdl(0)
    try:
        for name, fn in ops:
            out[name] = {"us": _time(fn, runner.stream, reps, iters)}
            for t, v in zip(state, snap):  # undo accumulations before the next op
                t.copy_(v)
    finally:
        lib().mq_set_pdl(pdl)
    torch.cuda.synchronize(runner.device)
    dims = [runner.g.feature_dim] + [int(w.shape[1]) for w in runner.model.weights]
    models = op_models(counts, dims, runner.tw.sw.fanouts, runner.Q, runner.cache is not None,
                       dm.num_params, runner.g.num_classes, runner.g.feature_dim)
    for name, rec in out.items():
        md = models.get(name, {})
        rec.update(md)
        sec = rec["us"] * 1e-6
        if md.get("bytes"):
            rec["gbps"] = md["bytes"] / sec / 1e9
        if md.get("sector_bytes"):
            rec["sector_gbps"] = md["sector_bytes"] / sec / 1e9
        if md.get("flops"):
            rec["tflops"] = md["flops"] / sec / 1e12
    return {"counts": counts, "ops": out}
