"""Drop-in SAGE numerics API backed by the CUDA kernels.

Mirrors ``mqpipe/nn.py``:

* ``ModelState``/``init_model`` — ``nn.py:19-71`` (Glorot uniform drawn with the
  reference's own NumPy generator, so weights are identical for a seed)
* ``forward``/``sage_forward``  — ``nn.py:116-138``
* ``batch_loss``                — ``nn.py:141-156``
* ``backward``                  — ``nn.py:159-180``
* ``loss_and_grads``            — ``nn.py:183-188``
* ``adam_step``/``sgd_step``    — ``nn.py:191-215``
* ``accuracy``                  — ``nn.py:253-256``

Parameters live in one flat fp32 device buffer (``engine.DeviceModel``);
``weights``, ``m`` and ``v`` are views into it.  Non-finite results raise
``FloatingPointError`` like the reference (``nn.py:74-76``).
"""

from __future__ import annotations

import numpy as np
import torch

from ._lib import lib, ptr
from .engine import DeviceModel, current_stream
from .graph import round_up

ADAM_BETA1 = 0.9
ADAM_BETA2 = 0.999
ADAM_EPS = 1e-8


class ModelState:
    """Weights plus Adam moments for one replica (flat device storage)."""

    def __init__(self, weights, arch: str = "sage", learning_rate: float = 0.001,
                 step_count: int = 0, m=None, v=None, device=None):
        if arch not in ("sage", "gcn"):
            raise ValueError(f"unknown arch {arch!r}")
        dev = torch.device(device or (weights[0].device if isinstance(weights[0], torch.Tensor)
                                      and weights[0].is_cuda else "cuda"))
        self.arch = arch
        self.dev = DeviceModel(weights, learning_rate, dev, step_count, m, v)

    # reference-compatible views
    @property
    def weights(self):
        return [self.dev.weight(i) for i in range(self.dev.num_layers)]

    @property
    def m(self):
        return [self.dev.view(self.dev.flat_m, i) for i in range(self.dev.num_layers)]

    @property
    def v(self):
        return [self.dev.view(self.dev.flat_v, i) for i in range(self.dev.num_layers)]

    @property
    def learning_rate(self):
        return self.dev.learning_rate

    @learning_rate.setter
    def learning_rate(self, lr):
        self.dev.learning_rate = float(lr)

    @property
    def step_count(self) -> int:
        return self.dev.host_steps

    @property
    def dtype(self):
        return torch.float32

    @property
    def device(self):
        return self.dev.device

    def copy(self) -> "ModelState":
        return ModelState([w.clone() for w in self.weights], self.arch, self.learning_rate,
                          self.step_count, [m.clone() for m in self.m],
                          [v.clone() for v in self.v], device=self.device)

    def to_numpy(self):
        return ([w.cpu().numpy() for w in self.weights], [m.cpu().numpy() for m in self.m],
                [v.cpu().numpy() for v in self.v])


def glorot_weights(feature_dim, hidden_dim, num_classes, num_layers=2, seed=0, arch="sage"):
    """Same draws as nn.py:56-71 (NumPy default_rng(seed); SAGE fan-in 2x)."""
    rng = np.random.default_rng(seed)
    dims = [feature_dim] + [hidden_dim] * (num_layers - 1) + [num_classes]
    out = []
    for l in range(num_layers):
        fan_in, fan_out = dims[l] * (2 if arch == "sage" else 1), dims[l + 1]
        limit = np.sqrt(6.0 / (fan_in + fan_out))
        out.append(rng.uniform(-limit, limit, size=(fan_in, fan_out)).astype(np.float32))
    return out


def init_model(feature_dim: int, hidden_dim: int, num_classes: int, num_layers: int = 2,
               arch: str = "sage", seed: int = 0, learning_rate: float = 0.001,
               dtype=np.float32, device=None) -> ModelState:
    if np.dtype(dtype) != np.float32:
        raise NotImplementedError("the device path trains in float32 (nn.py default)")
    if arch not in ("sage", "gcn"):
        raise ValueError(f"unknown arch {arch!r}")
    w = glorot_weights(feature_dim, hidden_dim, num_classes, num_layers, seed, arch=arch)
    return ModelState(w, arch=arch, learning_rate=learning_rate, device=device)


def _check(state: ModelState, name: str):
    flag = int(state.dev.nonfinite.item())
    if flag & 1:
        state.dev.nonfinite.zero_()
        raise FloatingPointError(f"{name} contains NaN or Inf")
    if flag & 2:
        state.dev.nonfinite.zero_()
        raise RuntimeError("optimizer step counter overflow")


def _finite_or_raise(name, t):
    if not bool(torch.isfinite(t).all()):
        raise FloatingPointError(f"{name} contains NaN or Inf")


def _pitched(x: torch.Tensor, ld: int) -> torch.Tensor:
    """Copy [n, d] into a zero-padded [n, ld] buffer (16-byte aligned rows)."""
    n, d = x.shape
    if x.is_contiguous() and d == ld:
        return x
    out = torch.zeros((max(n, 1), ld), dtype=torch.float32, device=x.device)
    out[:n, :d] = x
    return out


def _tc_linear_ok(d_in: int, d_out: int) -> bool:
    """The per-op SAGE transform runs on the tensor cores (tcgen05 3xTF32, the
    aggregate-first kernels of the fused step) where their shape rules allow;
    otherwise the fp32 split-K FFMA GEMM."""
    return (lib().mq_get_gemm_backend() == 1 and d_in >= 4 and d_in % 4 == 0
            and d_out <= 256)


def sage_forward(batch, state: ModelState, return_cache: bool = False):
    """Per layer: agg = segment-mean SpMM, z = [agg | h_dst] W, ReLU except last."""
    dev = state.device
    stream = current_stream(dev)
    h = batch.features.to(device=dev, dtype=torch.float32)
    cache = {"inputs": [], "pre": []}
    L = len(batch.layers)
    for l, blk in enumerate(batch.layers):
        d_in = int(h.shape[1])
        ld = round_up(d_in, 4)
        hp = _pitched(h, ld)
        nd = blk.num_dst
        nd_dev = torch.tensor([nd], dtype=torch.int32, device=dev)
        agg = torch.zeros((max(nd, 1), ld), dtype=torch.float32, device=dev)
        lib().mq_spmm_fwd(ptr(blk.row_ptr), ptr(blk.cols), ptr(blk.values), ptr(nd_dev), nd,
                          ptr(hp), ld, d_in, ptr(agg), ld, stream)
        W = state.weights[l]
        d_out = int(W.shape[1])
        z = torch.empty((max(nd, 1), d_out), dtype=torch.float32, device=dev)
        r = torch.empty((max(nd, 1), d_out), dtype=torch.float32, device=dev) if l < L - 1 else None
        if _tc_linear_ok(d_in, d_out):  # z = [agg | h_dst] W on tcgen05, then relu
            part = torch.empty(int(lib().mq_full_linear_cat_part_floats(nd, d_out)),
                               dtype=torch.float32, device=dev)
            lib().mq_full_linear_cat(ptr(agg), ld, ptr(hp), ld, nd, d_in, ptr(W), d_out, ptr(z),
                                     d_out, 0, ptr(part), stream)
            if r is not None:
                lib().mq_relu(ptr(z), ptr(r), nd * d_out, stream)
        else:
            scr = torch.empty(int(lib().mq_linear_scratch_bytes(nd, d_in, d_out)) // 4 + 1,
                              dtype=torch.float32, device=dev)
            lib().mq_sage_linear_fwd(ptr(agg), ld, ptr(hp), ld, ptr(nd_dev), nd, d_in, ptr(W),
                                     d_out, ptr(z), d_out, ptr(r), d_out, ptr(scr), stream)
        cache["inputs"].append((hp, agg, blk, nd_dev, d_in))
        cache["pre"].append(z[:nd])
        h = r[:nd] if l < L - 1 else z[:nd]
    _finite_or_raise("sage_forward output", h)
    return (h, cache) if return_cache else h


def gcn_forward(batch, state: ModelState, return_cache: bool = False):
    """GCN arm (nn.py:102-113): agg = block_apply(effective values), z = agg W,
    ReLU except the last layer."""
    dev = state.device
    stream = current_stream(dev)
    h = batch.features.to(device=dev, dtype=torch.float32)
    cache = {"inputs": [], "pre": []}
    L = len(batch.layers)
    for l, blk in enumerate(batch.layers):
        d_in = int(h.shape[1])
        ld = round_up(d_in, 4)
        hp = _pitched(h, ld)
        nd = blk.num_dst
        nd_dev = torch.tensor([nd], dtype=torch.int32, device=dev)
        agg = torch.zeros((max(nd, 1), ld), dtype=torch.float32, device=dev)
        lib().mq_spmm_fwd(ptr(blk.row_ptr), ptr(blk.cols), ptr(blk.values), ptr(nd_dev), nd,
                          ptr(hp), ld, d_in, ptr(agg), ld, stream)
        W = state.weights[l]
        d_out = int(W.shape[1])
        z = torch.empty((max(nd, 1), d_out), dtype=torch.float32, device=dev)
        r = torch.empty((max(nd, 1), d_out), dtype=torch.float32, device=dev) if l < L - 1 else None
        scr = torch.empty(int(lib().mq_linear_scratch_bytes(nd, d_in, d_out)) // 4 + 1,
                          dtype=torch.float32, device=dev)
        lib().mq_gcn_linear_fwd(ptr(agg), ld, ptr(nd_dev), nd, d_in, ptr(W), d_out, ptr(z), d_out,
                                ptr(r), d_out, ptr(scr), stream)
        cache["inputs"].append((hp, agg, blk, nd_dev, d_in))
        cache["pre"].append(z[:nd])
        h = r[:nd] if l < L - 1 else z[:nd]
    _finite_or_raise("gcn_forward output", h)
    return (h, cache) if return_cache else h


def forward(batch, state: ModelState, return_cache: bool = False):
    fn = sage_forward if state.arch == "sage" else gcn_forward
    return fn(batch, state, return_cache=return_cache)


def batch_loss(logits: torch.Tensor, labels):
    """Summed softmax-CE and dlogits (nn.py:141-156)."""
    dev = logits.device
    n, C = logits.shape
    lab = torch.as_tensor(labels).to(device=dev, dtype=torch.int32).contiguous()
    logits = logits.contiguous().to(torch.float32)
    n_dev = torch.tensor([n], dtype=torch.int32, device=dev)
    dl = torch.empty((max(n, 1), C), dtype=torch.float32, device=dev)
    loss = torch.zeros(1, dtype=torch.float64, device=dev)
    bad = torch.zeros(1, dtype=torch.int32, device=dev)
    lib().mq_softmax_ce(ptr(logits), C, ptr(lab), ptr(n_dev), n, C, ptr(dl), C, ptr(loss), ptr(bad),
                        current_stream(dev))
    if int(bad.item()):
        raise FloatingPointError("batch_loss contains NaN or Inf")
    return float(loss.item()), dl[:n]


def _tc_weight_grad(agg, hp, ld, nd_dev, nd, d_in, dz, lddz, d_out, dW, stream):
    """dW = [agg | h]^T dz (nn.py:167-170) through the aggregate-first weight
    gradient kernel (tcgen05, split-K partials [S][2 d_in][d_out]) and one
    fixed-order reduction into dW."""
    from ._lib import GradSrc
    import ctypes as C
    dev = dW.device
    parts = torch.empty(int(lib().mq_sage_af_dw_parts_bytes(d_in, d_out)) // 4 + 1,
                        dtype=torch.float32, device=dev)
    nparts = torch.zeros(1, dtype=torch.int32, device=dev)
    dzc = dz if (dz.is_contiguous() and lddz % 4 == 0) else None
    if dzc is None:  # a 16-byte-aligned pitch for the tensor-map operand
        lp = (d_out + 3) // 4 * 4
        dzc = torch.zeros((max(nd, 1), lp), dtype=torch.float32, device=dev)
        dzc[:nd, :d_out] = dz[:nd, :d_out]
        lddz = lp
    ones = torch.ones((max(nd, 1), lddz), dtype=torch.float32, device=dev)
    lib().mq_sage_linear_af_bwd(ptr(agg), ld, ptr(hp), ld, ptr(nd_dev), nd, d_in, ptr(dzc), lddz,
                                ptr(ones), lddz, d_out, ptr(parts), ptr(nparts), stream)
    src = GradSrc()
    seg = src.seg[0]
    seg.part = ptr(parts)
    seg.nparts_dev = ptr(nparts)
    seg.stride = 2 * d_in * d_out
    seg.offset = 0
    seg.size = 2 * d_in * d_out
    seg.nparts = 0
    seg.kind = 0
    src.nseg = 1
    lib().mq_grad_reduce(C.byref(src), ptr(dW), 2 * d_in * d_out, ptr(dW), stream)


def _gcn_backward(batch, state: ModelState, cache, dlogits: torch.Tensor) -> list:
    """GCN arm of nn.py:159-180: dW = agg^T dz, dh = block_apply_t(dz W^T)."""
    dev = state.device
    stream = current_stream(dev)
    L = len(batch.layers)
    grads = [None] * L
    dz = dlogits.contiguous().to(torch.float32)
    lddz = int(dz.shape[1])
    zero = torch.zeros(1, dtype=torch.int32, device=dev)
    for l in range(L - 1, -1, -1):
        hp, agg, blk, nd_dev, d_in = cache["inputs"][l]
        ld = int(hp.shape[1])
        nd = blk.num_dst
        W = state.weights[l]
        d_out = int(W.shape[1])
        dW = torch.empty_like(W)
        scr = torch.empty(int(lib().mq_linear_scratch_bytes(nd, d_in, d_out)) // 4 + 1,
                          dtype=torch.float32, device=dev)
        dt = (torch.zeros((max(nd, 1), 2 * d_in), dtype=torch.float32, device=dev)
              if l > 0 else None)
        lib().mq_gcn_linear_bwd(ptr(agg), ld, ptr(nd_dev), nd, d_in, ptr(W), d_out, ptr(dz), lddz,
                                ptr(dW), ptr(dt), 2 * d_in, ptr(scr), stream)
        grads[l] = dW
        if l > 0:
            ns = blk.num_src
            counts = torch.tensor([ns, blk.nnz], dtype=torch.int32, device=dev)
            dh = torch.empty((max(ns, 1), ld), dtype=torch.float32, device=dev)
            # no self half: the init pass sees zero dst rows (every dh row starts at 0)
            lib().mq_spmm_bwd(ptr(blk.rows), ptr(blk.cols), ptr(blk.values), ptr(counts), blk.nnz,
                              ptr(zero), ns, ptr(dt), 2 * d_in, d_in, ptr(hp), ld, ptr(dh), ld,
                              stream)
            dz, lddz = dh, ld
    for g in grads:
        _finite_or_raise("backward", g)
    return grads


def backward(batch, state: ModelState, cache, dlogits: torch.Tensor) -> list:
    """Weight gradients, last layer first (nn.py:159-180)."""
    if state.arch == "gcn":
        return _gcn_backward(batch, state, cache, dlogits)
    dev = state.device
    stream = current_stream(dev)
    L = len(batch.layers)
    grads = [None] * L
    dz = dlogits.contiguous().to(torch.float32)
    lddz = int(dz.shape[1])
    for l in range(L - 1, -1, -1):
        hp, agg, blk, nd_dev, d_in = cache["inputs"][l]
        ld = int(hp.shape[1])
        nd = blk.num_dst
        W = state.weights[l]
        d_out = int(W.shape[1])
        dW = torch.empty_like(W)
        scr = torch.empty(int(lib().mq_linear_scratch_bytes(nd, d_in, d_out)) // 4 + 1,
                          dtype=torch.float32, device=dev)
        dt = torch.empty((max(nd, 1), 2 * d_in), dtype=torch.float32, device=dev) if l > 0 else None
        if _tc_linear_ok(d_in, d_out) and nd > 0:
            # dW = [agg | h_dst]^T dz on tcgen05 (deferred split-K partials,
            # reduced in fixed order); dz is already masked, so the kernel's
            # (act > 0) mask gets ones
            _tc_weight_grad(agg, hp, ld, nd_dev, nd, d_in, dz, lddz, d_out, dW, stream)
            if dt is not None:  # dt = dz W^T: K = d_out, the FFMA GEMM
                lib().mq_sage_linear_dt(ptr(nd_dev), nd, d_in, ptr(W), d_out, ptr(dz), lddz,
                                        ptr(dt), 2 * d_in, ptr(scr), stream)
        else:
            lib().mq_sage_linear_bwd(ptr(agg), ld, ptr(hp), ld, ptr(nd_dev), nd, d_in, ptr(W),
                                     d_out, ptr(dz), lddz, ptr(dW), ptr(dt), 2 * d_in, ptr(scr),
                                     stream)
        grads[l] = dW
        if l > 0:
            ns = blk.num_src
            counts = torch.tensor([ns, blk.nnz], dtype=torch.int32, device=dev)
            dh = torch.empty((max(ns, 1), ld), dtype=torch.float32, device=dev)
            lib().mq_spmm_bwd(ptr(blk.rows), ptr(blk.cols), ptr(blk.values), ptr(counts), blk.nnz,
                              ptr(nd_dev), ns, ptr(dt), 2 * d_in, d_in, ptr(hp), ld, ptr(dh), ld,
                              stream)
            dz, lddz = dh, ld
    for g in grads:
        _finite_or_raise("backward", g)
    return grads


def loss_and_grads(batch, state: ModelState):
    logits, cache = forward(batch, state, return_cache=True)
    loss, dlogits = batch_loss(logits, batch.target_labels)
    grads = backward(batch, state, cache, dlogits)
    return loss, grads, logits


def _flat_grad(state: ModelState, grads):
    g = state.dev.flat_g
    for i, gi in enumerate(grads):
        state.dev.grad(i).copy_(torch.as_tensor(gi).to(device=g.device, dtype=torch.float32)
                                if not isinstance(gi, torch.Tensor) else gi.to(torch.float32))
    return g


def adam_step(state: ModelState, grads: list) -> ModelState:
    """Bias-corrected Adam, bit-identical op order to nn.py:191-206."""
    _flat_grad(state, grads)
    d = state.dev
    d.ensure_bias(d.host_steps + 1)
    lib().mq_adam(ptr(d.flat_w), ptr(d.flat_m), ptr(d.flat_v), ptr(d.flat_g), None, 1.0,
                  d.num_params, ptr(d.step_dev), ptr(d.bias), d.bias_len, ptr(d.lr_dev),
                  ptr(d.nonfinite), None, current_stream(d.device))
    d.host_steps += 1
    _check(state, "adam_step")
    return state


def sgd_step(state: ModelState, grads: list) -> ModelState:
    _flat_grad(state, grads)
    d = state.dev
    lib().mq_sgd(ptr(d.flat_w), ptr(d.flat_g), None, 1.0, d.num_params, ptr(d.step_dev), ptr(d.lr_dev),
                 ptr(d.nonfinite), None, current_stream(d.device))
    d.host_steps += 1
    _check(state, "sgd_step")
    return state


def accuracy(logits, labels) -> float:
    logits = torch.as_tensor(logits)
    if logits.shape[0] == 0:
        return 0.0
    lab = torch.as_tensor(labels, device=logits.device)
    return float((logits.argmax(dim=1) == lab.long()).float().mean().item())


# ------------------------------------------------------- full-graph evaluation
class _EvalWorkspace:
    """Per-(graph, layer widths) buffers of full_forward, reused across epochs."""

    def __init__(self, g, dims):
        dev = g.device
        n = max(g.num_nodes, 1)
        self.dims = tuple(dims)
        self.y, self.part, self.out, self.scratch = [], [], [], []
        for l in range(len(dims) - 1):
            d_out = dims[l + 1]
            last = l == len(dims) - 2
            self.y.append(torch.empty((n, 2 * d_out), dtype=torch.float32, device=dev))
            self.part.append(torch.empty(int(lib().mq_full_transform_part_floats(n, d_out)),
                                         dtype=torch.float32, device=dev))
            self.out.append(torch.empty((n, d_out if last else round_up(d_out, 4)),
                                        dtype=torch.float32, device=dev))
            self.scratch.append(torch.empty(
                int(lib().mq_full_agg_scratch_bytes(g.num_arcs, d_out)), dtype=torch.uint8,
                device=dev))
        # the transform scratch is only live inside one layer: share the largest
        big = max(self.part, key=lambda t: t.numel())
        self.part = [big] * len(self.part)
        self.correct = torch.zeros(1, dtype=torch.int64, device=dev)


def _eval_ws(g, dims):
    ws = getattr(g, "_eval_ws", None)
    if ws is None or ws.dims != tuple(dims):
        ws = _EvalWorkspace(g, dims)
        g._eval_ws = ws
    return ws


def full_forward(g, state: ModelState) -> torch.Tensor:
    """Exact whole-graph forward pass (nn.py:218-250, sage arm) on the device.

    Per layer: Y = h [W_top | W_bot] (tcgen05 3xTF32 GEMM over every node),
    then z[v] = f32(1/deg v) * sum_{v->u} Y_top[u] + Y_bot[v] over the
    loop-stripped CSR (nn.py:236-243), ReLU except after the last layer.
    Returns logits [n, num_classes] (fp32 re-association of the reference;
    DESIGN.md §5 tolerance)."""
    if state.arch != "sage":
        raise ValueError("full_forward implements the sage arch")
    dev = g.device
    stream = current_stream(dev)
    dims = [g.feature_dim] + [int(w.shape[1]) for w in state.weights]
    if int(state.weights[0].shape[0]) != 2 * g.feature_dim:
        raise ValueError("model input width does not match the graph's features")
    g.require_full_table("full_forward")
    ws = _eval_ws(g, dims)
    n = g.num_nodes
    h, ldh = g.features, g.pitch
    L = len(state.weights)
    for l, W in enumerate(state.weights):
        d_in, d_out = dims[l], dims[l + 1]
        lib().mq_full_transform(ptr(h), ldh, n, d_in, ptr(W), d_out, ptr(ws.y[l]),
                                ptr(ws.part[l]), stream)
        out = ws.out[l]
        lib().mq_full_aggregate(ptr(g.row_off), ptr(g.col), n, g.num_arcs, ptr(ws.y[l]),
                                2 * d_out, d_out, 0 if l == L - 1 else 1, ptr(out),
                                int(out.shape[1]), ptr(ws.scratch[l]), stream)
        h, ldh = out, int(out.shape[1])
    logits = ws.out[-1][:n]
    _finite_or_raise("full_forward", logits)
    return logits


def _full_fits(g, state: ModelState) -> bool:
    """full_forward's workspace (cached per graph) fits in free HBM with a margin."""
    dims = [g.feature_dim] + [int(w.shape[1]) for w in state.weights]
    ws = getattr(g, "_eval_ws", None)
    if ws is not None and ws.dims == tuple(dims):
        return True
    n = max(g.num_nodes, 1)
    need = 0
    for l in range(len(dims) - 1):
        d_out = dims[l + 1]
        need += 4 * n * (3 * d_out + 4)
        need += 4 * int(lib().mq_full_transform_part_floats(n, d_out))
        need += int(lib().mq_full_agg_scratch_bytes(g.num_arcs, d_out))
    free, _ = torch.cuda.mem_get_info(g.device)
    return need < 0.8 * free


def evaluate(g, state: ModelState, mask, chunk: int = 1 << 20) -> float:
    """Accuracy over the nodes selected by ``mask`` (the reference driver's
    evaluate, bench.py:82-87: full_forward + accuracy), computed lean:

    * hidden layers transform-first with the bottom half accumulated in place:
      out = h W_bot, Y_top = h W_top, out[v] = relu(inv_v * sum Y_top[u] + out[v])
      (two n x d_out buffers instead of n x 2 d_out plus n x d_out);
    * the last layer aggregate-first for the evaluated rows only, in chunks:
      agg_i = inv_v * sum h[u] (the reference's own agg row), logits =
      [agg | h_v] W, argmax against the label — no n x C logits.
    Same numerics as full_forward up to fp32 re-association."""
    idx = np.flatnonzero(np.asarray(mask))
    if idx.size == 0:
        return 0.0
    if state.arch != "sage":
        raise ValueError("evaluate implements the sage arch")
    if _full_fits(g, state):  # the full-graph form is faster when it fits
        logits = full_forward(g, state)
        ws = g._eval_ws
        ids = torch.as_tensor(idx.astype(np.int32)).to(g.device)
        ws.correct.zero_()
        lib().mq_accuracy(ptr(logits), int(logits.stride(0)), int(logits.shape[1]),
                          ptr(g.labels), ptr(ids), int(ids.numel()), ptr(ws.correct),
                          current_stream(g.device))
        return int(ws.correct.item()) / idx.size
    dev = g.device
    stream = current_stream(dev)
    lb = lib()
    dims = [g.feature_dim] + [int(w.shape[1]) for w in state.weights]
    if int(state.weights[0].shape[0]) != 2 * g.feature_dim:
        raise ValueError("model input width does not match the graph's features")
    n, L = g.num_nodes, len(state.weights)
    f32 = dict(dtype=torch.float32, device=dev)
    g.require_full_table("evaluate")
    h, ldh = g.features, g.pitch
    keep = []
    for l in range(L - 1):
        d_in, d_out = dims[l], dims[l + 1]
        W = state.weights[l]
        ld_out = round_up(d_out, 4)
        out = torch.zeros((max(n, 1), ld_out), **f32)
        ytop = torch.empty((max(n, 1), d_out), **f32)
        part = torch.empty(int(lb.mq_full_transform_part_floats(n, d_out)) + 1, **f32)
        lb.mq_full_transform_half(ptr(h), ldh, n, d_in, ptr(W), d_out, ptr(ytop), d_out,
                                  ptr(part), stream)
        lb.mq_full_transform_half(ptr(h), ldh, n, d_in, W.data_ptr() + 4 * d_in * d_out, d_out,
                                  ptr(out), ld_out, ptr(part), stream)
        scr = torch.empty(int(lb.mq_full_agg_scratch_bytes(g.num_arcs, d_out)), dtype=torch.uint8,
                          device=dev)
        lb.mq_full_aggregate_inplace(ptr(g.row_off), ptr(g.col), n, g.num_arcs, ptr(ytop), d_out,
                                     d_out, 1, ptr(out), ld_out, ptr(scr), stream)
        del ytop, part, scr
        keep = [out]  # the previous layer's output is no longer needed
        h, ldh = out, ld_out
    # last layer, aggregate-first over the evaluated rows: their means in one
    # full-graph pass restricted to them (hubs split across warps), then
    # logits = [agg | h_v] W in chunks, argmax against the label
    d_in, C = dims[L - 1], dims[L]
    W = state.weights[L - 1]
    ids_all = torch.as_tensor(idx.astype(np.int32)).to(dev)
    correct = torch.zeros(1, dtype=torch.int64, device=dev)
    if d_in % 4:  # (a 1-layer model on unpadded features) full logits, then argmax
        logits_all = full_forward(g, state)
        lb.mq_accuracy(ptr(logits_all), int(logits_all.stride(0)), C, ptr(g.labels), ptr(ids_all),
                       int(ids_all.numel()), ptr(correct), stream)
        return int(correct.item()) / idx.size
    ldi = round_up(d_in, 4)
    sel = torch.full((max(n, 1),), -1, dtype=torch.int32, device=dev)
    sel[ids_all.long()] = torch.arange(idx.size, dtype=torch.int32, device=dev)
    agg = torch.zeros((idx.size, ldi), **f32)
    scr = torch.empty(int(lb.mq_full_agg_scratch_bytes(g.num_arcs, d_in)), dtype=torch.uint8,
                      device=dev)
    lb.mq_full_aggregate_rows(ptr(g.row_off), ptr(g.col), n, g.num_arcs, ptr(h), ldh, d_in,
                              ptr(sel), ptr(agg), ldi, ptr(scr), stream)
    del scr, sel
    cap = min(chunk, idx.size)
    logits = torch.empty((cap, C), **f32)
    part = torch.empty(int(lb.mq_full_linear_cat_part_floats(cap, C)) + 1, **f32)
    for lo in range(0, idx.size, cap):
        m = min(cap, idx.size - lo)
        ids = ids_all[lo:lo + m]
        hv = h.index_select(0, ids.long())
        lb.mq_full_linear_cat(ptr(agg[lo:lo + m]), ldi, ptr(hv), ldh, m, d_in, ptr(W), C,
                              ptr(logits), C, 0, ptr(part), stream)
        _finite_or_raise("evaluate logits", logits[:m])
        lb.mq_accuracy_rows(ptr(logits), C, C, ptr(g.labels), ptr(ids), m, ptr(correct), stream)
    del keep
    return int(correct.item()) / idx.size
