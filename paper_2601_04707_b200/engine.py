"""Preallocated device workspaces for one training step and its CUDA graph.

Every buffer of the per-iteration path is sized
once from host-side upper bounds, so a whole step — batch setup, L hops of
sample + relabel, feature gather, forward, loss, backward, optimizer — is a
fixed sequence of C-ABI launches with no host synchronisation and can be
captured into one CUDA graph.  Counts that only the device knows (frontier
sizes, nnz) travel as device scalars.

Bounds for batch B and per-hop fanouts f_h (hop 0 at the seeds):
  n_dst_0 = B,  n_src_h = min(n_dst_h (1 + f_h), n_dst_h + |V|),
  n_dst_{h+1} = n_src_h,  nnz_h <= n_dst_h f_h.
Layer l (bottom-up) consumes hop L-1-l.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from ._lib import GradSrc, lib, ptr
from .graph import DeviceGraph, round_up


@dataclass
class HopBounds:
    fanout: int
    n_dst_max: int
    n_src_max: int

    @property
    def nnz_max(self) -> int:
        return self.n_dst_max * self.fanout


def hop_bounds(batch_size: int, fanouts, num_nodes: int) -> list:
    out = []
    nd = batch_size
    for f in fanouts:
        ns = min(nd * (1 + f), nd + num_nodes)
        out.append(HopBounds(int(f), nd, ns))
        nd = ns
    return out


class HopBuffers:
    """Device outputs of one hop of sample + relabel (one Block)."""

    def __init__(self, b: HopBounds, device):
        i32 = dict(dtype=torch.int32, device=device)
        self.bounds = b
        self.nbr = torch.zeros(max(b.nnz_max, 1), **i32)
        self.cnt = torch.zeros(max(b.n_dst_max, 1), **i32)
        self.row_ptr = torch.zeros(b.n_dst_max + 1, **i32)
        self.rows = torch.zeros(max(b.nnz_max, 1), **i32)
        self.cols = torch.zeros(max(b.nnz_max, 1), **i32)
        self.vals = torch.zeros(max(b.nnz_max, 1), dtype=torch.float32, device=device)
        self.src_ids = torch.zeros(max(b.n_src_max, 1), **i32)
        self.counts = torch.zeros(2, **i32)  # [n_src, nnz]


class SampleWorkspace:
    """Targets + the hop chain (sample_node_wise, samplers.py:213-226)."""

    def __init__(self, g: DeviceGraph, fanouts, batch_size: int):
        if not fanouts:
            raise ValueError("need at least one hop")
        if any(f < 1 or f > 32 for f in fanouts):
            raise ValueError("fanouts must lie in [1, 32]")
        dev = g.device
        self.graph = g
        self.fanouts = tuple(int(f) for f in fanouts)
        self.batch_size = int(batch_size)
        self.bounds = hop_bounds(self.batch_size, self.fanouts, g.num_nodes)
        self.targets = torch.zeros(max(self.batch_size, 1), dtype=torch.int32, device=dev)
        self.n_targets = torch.zeros(1, dtype=torch.int32, device=dev)
        self.key = torch.zeros(3, dtype=torch.int32, device=dev)  # uint32 seed, epoch, batch
        self.hops = [HopBuffers(b, dev) for b in self.bounds]
        scr = max(int(lib().mq_relabel_scratch_bytes(b.n_dst_max, b.fanout)) for b in self.bounds)
        self.scratch = torch.zeros(scr, dtype=torch.uint8, device=dev)
        # node-indexed relabel tables, private to this workspace so replicas
        # sampling concurrently on different streams never share them
        self.dpos = torch.full((g.num_nodes,), -1, dtype=torch.int32, device=dev)
        self.first = torch.full((g.num_nodes,), 2 ** 31 - 1, dtype=torch.int32, device=dev)
        # this slot's transfer-stage outputs: gathered input rows and target labels
        self.x0 = torch.zeros((max(self.bounds[-1].n_src_max, 1), g.pitch), dtype=torch.float32,
                              device=dev)
        self.labels = torch.zeros(max(self.batch_size, 1), dtype=torch.int32, device=dev)

    # device scalars for hop h
    def n_dst_dev(self, h: int) -> torch.Tensor:
        return self.n_targets if h == 0 else self.hops[h - 1].counts[0:1]

    def dst(self, h: int) -> torch.Tensor:
        return self.targets if h == 0 else self.hops[h - 1].src_ids

    @property
    def input_ids(self) -> torch.Tensor:
        return self.hops[-1].src_ids

    @property
    def n_input_dev(self) -> torch.Tensor:
        return self.hops[-1].counts[0:1]

    def launch(self, cache, stream, *, seed=0, epoch=0, batch=0, key_on_device=False):
        g = self.graph
        L = lib()
        hot_arc = ptr(cache.hot_arc) if cache is not None else None
        hot_off = ptr(cache.hot_off) if cache is not None else None
        key = ptr(self.key) if key_on_device else None
        for h, (hb, b) in enumerate(zip(self.hops, self.bounds)):
            L.mq_sample_hop(ptr(g.row_off), ptr(g.col), hot_arc, hot_off, ptr(self.dst(h)),
                            ptr(self.n_dst_dev(h)), b.n_dst_max, b.fanout, seed & 0xFFFFFFFF,
                            epoch & 0xFFFFFFFF, batch & 0xFFFFFFFF, h, key, ptr(hb.nbr),
                            ptr(hb.cnt), stream)
            L.mq_relabel(ptr(self.dst(h)), ptr(self.n_dst_dev(h)), b.n_dst_max, ptr(hb.nbr),
                         ptr(hb.cnt), b.fanout, ptr(self.dpos), ptr(self.first), ptr(hb.row_ptr),
                         ptr(hb.rows), ptr(hb.cols), ptr(hb.vals), ptr(hb.src_ids),
                         ptr(hb.counts), ptr(self.scratch), stream)


class DeviceModel:
    """Flat fp32 parameters + Adam moments (ModelState, nn.py:19-53)."""

    def __init__(self, weights, learning_rate: float, device, step_count: int = 0,
                 m=None, v=None, bias_len: int = 1 << 16):
        self.shapes = [tuple(int(x) for x in w.shape) for w in weights]
        self.offsets = np.cumsum([0] + [a * b for a, b in self.shapes]).tolist()
        n = self.offsets[-1]
        self.num_params = n
        self.device = device
        # float32(learning_rate) in device memory: the optimizer kernels read it
        # per launch, so captured step graphs follow learning-rate changes
        self.lr_dev = torch.zeros(1, dtype=torch.float32, device=device)
        self._lr = None
        self.learning_rate = float(learning_rate)
        self.flat_w = torch.zeros(n, dtype=torch.float32, device=device)
        self.flat_m = torch.zeros(n, dtype=torch.float32, device=device)
        self.flat_v = torch.zeros(n, dtype=torch.float32, device=device)
        self.flat_g = torch.zeros(n, dtype=torch.float32, device=device)
        for i, w in enumerate(weights):
            self.weight(i).copy_(_t(w, device))
            if m is not None:
                self.view(self.flat_m, i).copy_(_t(m[i], device))
            if v is not None:
                self.view(self.flat_v, i).copy_(_t(v[i], device))
        # [update count t, optimizer arrival counter] (mqgnn.h mq_adam)
        self.step_dev = torch.tensor([step_count, 0], dtype=torch.int32, device=device)
        self.nonfinite = torch.zeros(1, dtype=torch.int32, device=device)
        self.bias, self.bias_len = _bias_table(max(bias_len, BIAS_SATURATED), device)
        self.host_steps = step_count

    def ensure_bias(self, steps: int):
        """The bias-correction table is allocated once and never replaced:
        captured graphs hold its pointer.  It ends at the saturated row
        (1.0f, 1.0f), which the kernel reads for every later step — exactly
        float32(1 - beta**t) there (mqgnn.h mq_adam)."""
        return None

    @property
    def learning_rate(self) -> float:
        return self._lr

    @learning_rate.setter
    def learning_rate(self, lr: float):
        lr = float(lr)
        if lr != self._lr:
            self._lr = lr
            # synchronous: graphs replayed later on any stream read the new value
            self.lr_dev.fill_(float(np.float32(lr)))
            if self.lr_dev.is_cuda:
                torch.cuda.synchronize(self.lr_dev.device)

    def view(self, flat, i):
        a, b = self.shapes[i]
        return flat[self.offsets[i]:self.offsets[i + 1]].view(a, b)

    def weight(self, i):
        return self.view(self.flat_w, i)

    def grad(self, i):
        return self.view(self.flat_g, i)

    @property
    def num_layers(self):
        return len(self.shapes)

    @property
    def lr32(self) -> float:
        return float(np.float32(self.learning_rate))


# float32(1 - 0.999**t) == 1.0f from t ~ 17.3k on; past this length both
# columns are exactly 1.0f, so clamping t to the last row is exact
BIAS_SATURATED = 1 << 16


def _bias_table(steps: int, device):
    """float32(1 - beta1**t), float32(1 - beta2**t) for t = 1..steps, computed
    with Python floats exactly as nn.py:202-203 does."""
    tab = np.empty((steps, 2), dtype=np.float32)
    tab[:, 0] = np.array([1 - 0.9 ** k for k in range(1, steps + 1)],
                         dtype=np.float64).astype(np.float32)
    tab[:, 1] = np.array([1 - 0.999 ** k for k in range(1, steps + 1)],
                         dtype=np.float64).astype(np.float32)
    if not (tab[-1] == 1.0).all():
        raise ValueError("bias table must reach the saturated (1, 1) row")
    return torch.as_tensor(tab.reshape(-1), device=device), steps


def _t(a, device):
    if isinstance(a, torch.Tensor):
        return a.to(device=device, dtype=torch.float32)
    return torch.as_tensor(np.asarray(a, dtype=np.float32), device=device)


class TrainWorkspace:
    """Activation / gradient buffers of one SAGE step.

    The per-batch inputs (hop CSR blocks, gathered features ``x0``, labels)
    live in a SampleWorkspace "slot"; every launch method takes the slot it
    consumes so two slots can be double-buffered (prep of batch k+1 while
    batch k trains)."""

    def __init__(self, sw: SampleWorkspace, dims, num_classes: int):
        g = sw.graph
        dev = g.device
        L = len(sw.fanouts)
        if len(dims) != L + 1:
            raise ValueError("dims must list input, hidden..., classes")
        self.sw = sw
        self.dims = list(dims)
        self.L = L
        self.C = num_classes
        f32 = dict(dtype=torch.float32, device=dev)
        self.ld_in = [g.pitch] + [round_up(d, 4) for d in self.dims[1:L]]
        self.agg, self.act, self.dt, self.dh = [], [None], [], []
        for l in range(L):
            b = sw.bounds[L - 1 - l]
            self.agg.append(torch.zeros((max(b.n_dst_max, 1), self.ld_in[l]), **f32))
            if l + 1 < L:
                self.act.append(torch.zeros((max(b.n_dst_max, 1), self.ld_in[l + 1]), **f32))
            if l > 0:
                self.dt.append(torch.zeros((max(b.n_dst_max, 1), 2 * self.dims[l]), **f32))
                self.dh.append(torch.zeros((max(b.n_src_max, 1), self.ld_in[l]), **f32))
            else:
                self.dt.append(None)
                self.dh.append(None)
        B = sw.batch_size
        self.logits = torch.zeros((max(B, 1), num_classes), **f32)
        self.dlogits = torch.zeros((max(B, 1), num_classes), **f32)
        self.loss = torch.zeros(1, dtype=torch.float64, device=dev)
        scr = max(int(lib().mq_linear_scratch_bytes(sw.bounds[L - 1 - l].n_dst_max,
                                                    self.dims[l], self.dims[l + 1]))
                  for l in range(L))
        self.scratch = torch.zeros(scr // 4 + 1, **f32)

    @property
    def x0(self):
        return self.sw.x0

    def h_in(self, l, sw=None):
        return (sw or self.sw).x0 if l == 0 else self.act[l]

    @staticmethod
    def launch_gather(sw: SampleWorkspace, cache, stream):
        """transfer_stage (runtime.py:127-143) + target labels (samplers.py:532)."""
        g = sw.graph
        b = sw.bounds[-1]
        g.gather_rows(sw.input_ids, sw.n_input_dev, b.n_src_max, sw.x0, g.pitch, stream,
                      cache=cache, hit_miss=cache.hit_miss if cache is not None else None)
        lib().mq_gather_labels(ptr(g.labels), ptr(sw.targets), ptr(sw.n_targets), sw.batch_size,
                               ptr(sw.labels), stream)

    def launch_forward(self, model: DeviceModel, stream, sw=None):
        sw = sw or self.sw
        L = self.L
        for l in range(L):
            h = L - 1 - l
            hb, b = sw.hops[h], sw.bounds[h]
            nd = sw.n_dst_dev(h)
            hin = self.h_in(l, sw)
            lib().mq_spmm_fwd(ptr(hb.row_ptr), ptr(hb.cols), ptr(hb.vals), ptr(nd), b.n_dst_max,
                              ptr(hin), self.ld_in[l], self.dims[l], ptr(self.agg[l]),
                              self.ld_in[l], stream)
            W = model.weight(l)
            if l + 1 < L:
                lib().mq_sage_linear_fwd(ptr(self.agg[l]), self.ld_in[l], ptr(hin), self.ld_in[l],
                                         ptr(nd), b.n_dst_max, self.dims[l], ptr(W),
                                         self.dims[l + 1], None, 0, ptr(self.act[l + 1]),
                                         self.ld_in[l + 1], ptr(self.scratch), stream)
            else:
                lib().mq_sage_linear_fwd(ptr(self.agg[l]), self.ld_in[l], ptr(hin), self.ld_in[l],
                                         ptr(nd), b.n_dst_max, self.dims[l], ptr(W),
                                         self.dims[l + 1], ptr(self.logits), self.C, None, 0,
                                         ptr(self.scratch), stream)

    def launch_loss(self, model: DeviceModel, stream, sw=None):
        sw = sw or self.sw
        lib().mq_softmax_ce(ptr(self.logits), self.C, ptr(sw.labels), ptr(sw.n_targets),
                            sw.batch_size, self.C, ptr(self.dlogits), self.C, ptr(self.loss),
                            ptr(model.nonfinite), stream)

    def launch_backward(self, model: DeviceModel, stream, sw=None):
        sw = sw or self.sw
        L = self.L
        dz, lddz = self.dlogits, self.C
        for l in range(L - 1, -1, -1):
            h = L - 1 - l
            hb, b = sw.hops[h], sw.bounds[h]
            nd = sw.n_dst_dev(h)
            hin = self.h_in(l, sw)
            d_in, d_out = self.dims[l], self.dims[l + 1]
            dt = self.dt[l]
            lib().mq_sage_linear_bwd(ptr(self.agg[l]), self.ld_in[l], ptr(hin), self.ld_in[l],
                                     ptr(nd), b.n_dst_max, d_in, ptr(model.weight(l)), d_out,
                                     ptr(dz), lddz, ptr(model.grad(l)), ptr(dt), 2 * d_in,
                                     ptr(self.scratch), stream)
            if l > 0:
                lib().mq_spmm_bwd(ptr(hb.rows), ptr(hb.cols), ptr(hb.vals), ptr(hb.counts),
                                  b.nnz_max, ptr(nd), b.n_src_max, ptr(dt), 2 * d_in, d_in,
                                  ptr(hin), self.ld_in[l], ptr(self.dh[l]), self.ld_in[l], stream)
                dz, lddz = self.dh[l], self.ld_in[l]

    @staticmethod
    def launch_optimizer(model: DeviceModel, optimizer: str, stream, grad64=None, scale=1.0,
                         src=None):
        """apply_update (racom.py:81-87): the gradient is model.flat_g resolved
        through the deferred split-K segments ``src`` (a _lib.GradSrc), or the
        all-reduced f64 window sum ``grad64``."""
        g32 = None if grad64 is not None else ptr(model.flat_g)
        g64 = ptr(grad64) if grad64 is not None else None
        psrc = C.byref(src) if (src is not None and grad64 is None) else None
        if optimizer == "adam":
            lib().mq_adam(ptr(model.flat_w), ptr(model.flat_m), ptr(model.flat_v), g32, g64, scale,
                          model.num_params, ptr(model.step_dev), ptr(model.bias), model.bias_len,
                          ptr(model.lr_dev), ptr(model.nonfinite), psrc, stream)
        elif optimizer == "sgd":
            lib().mq_sgd(ptr(model.flat_w), g32, g64, scale, model.num_params,
                         ptr(model.step_dev), ptr(model.lr_dev), ptr(model.nonfinite), psrc, stream)
        else:
            raise ValueError(f"unknown optimizer {optimizer!r}")


class FusedTrainWorkspace:
    """Buffers of the fused SAGE step (csrc/mq_fused.cu).

    Layers 0..L-2 run transform-first (Y = h [W_top | W_bot], then a
    d_out-wide aggregation); layer L-1 (the seeds' block) is the one-launch
    head (aggregate + transform + softmax-CE + its backward + deterministic
    dW).  Per layer l (hop h = L-1-l):
      Y[l], G[l]   (n_src_h x 2 d_{l+1})   transform output / its gradient
      act[l+1]     (n_dst_h x ld_{l+1})    relu output = next layer's input
      dh[l]        (n_src_h x ld_l)        gradient w.r.t. layer l's input, l >= 1
    The scatter targets (G[l], dh[L-1]) are cleared by the forward's
    aggregation kernels, so the step has no memset nodes.

    The input layer may instead run aggregate-first (``layer0="af"``; "auto"
    picks it when d_in <= 2 d_out and d_in % 4 == 0): agg0 = block_apply(x0)
    (mq_spmm_fwd, bit-exact), act1 = relu([agg0 | x0] W0) and its weight
    gradient [agg0 | x0]^T (dh1 * mask) on the tensor cores.  For narrow
    inputs (products-shaped 100-d) this reads n_dst rows instead of
    transforming every n_src row, and layer 0 needs no scatter (the input
    has no gradient)."""

    def __init__(self, sw: SampleWorkspace, dims, num_classes: int, layer0: str = "auto"):
        g = sw.graph
        dev = g.device
        L = len(sw.fanouts)
        if len(dims) != L + 1:
            raise ValueError("dims must list input, hidden..., classes")
        self.sw = sw
        self.dims = list(dims)
        self.L = L
        self.C = num_classes
        f32 = dict(dtype=torch.float32, device=dev)
        self.ld_in = [g.pitch] + [round_up(d, 4) for d in self.dims[1:L]]
        if layer0 not in ("auto", "tf", "af"):
            raise ValueError(f"layer0 must be auto, tf or af, not {layer0!r}")
        af_ok = (L >= 2 and self.dims[0] % 4 == 0 and self.dims[1] <= 256
                 and lib().mq_get_gemm_backend() == 1)
        if layer0 == "af" and not af_ok:
            raise ValueError("aggregate-first layer 0 needs d_in % 4 == 0, d_out <= 256, L >= 2 "
                             "and the tensor-core backend")
        self.af0 = af_ok and (layer0 == "af" or
                              (layer0 == "auto" and self.dims[0] <= 2 * self.dims[1]))
        self.Y, self.G, self.act, self.dh = [], [], [None] * (L + 1), [None] * L
        scr = 1
        for l in range(L - 1):
            b = sw.bounds[L - 1 - l]
            n2 = 2 * self.dims[l + 1]
            if l == 0 and self.af0:
                self.Y.append(None)
                self.G.append(None)
                self.agg0 = torch.zeros((max(b.n_dst_max, 1), self.ld_in[0]), **f32)
                self.af_part = torch.zeros(
                    int(lib().mq_sage_af_parts_bytes(b.n_dst_max, self.dims[1])) // 4 + 1, **f32)
                self.act[1] = torch.zeros((max(b.n_dst_max, 1), self.ld_in[1]), **f32)
                continue
            # Y, or (tensor-core backend) its deferred split-K partial tiles
            ny = max(b.n_src_max, 1) * n2
            ny = max(ny, int(lib().mq_sage_y_parts_bytes(b.n_src_max, self.dims[l + 1])) // 4)
            self.Y.append(torch.zeros(ny, **f32))
            self.G.append(torch.zeros((max(b.n_src_max, 1), n2), **f32))
            self.act[l + 1] = torch.zeros((max(b.n_dst_max, 1), self.ld_in[l + 1]), **f32)
            if l >= 1:
                self.dh[l] = torch.zeros((max(b.n_src_max, 1), self.ld_in[l]), **f32)
            scr = max(scr, int(lib().mq_sage_fused_scratch_bytes(b.n_src_max, self.dims[l],
                                                                  self.dims[l + 1])))
        if L > 1:
            b0 = sw.bounds[0]
            self.dh[L - 1] = torch.zeros((max(b0.n_src_max, 1), self.ld_in[L - 1]), **f32)
        self.scratch = torch.zeros(scr // 4 + 1, **f32)
        hb = int(lib().mq_sage_head_scratch_bytes(sw.batch_size, self.dims[L - 1], num_classes))
        self.head_scratch = torch.zeros(hb // 4 + 1, **f32)  # zeroed once: completion counter
        self.loss = torch.zeros(1, dtype=torch.float64, device=dev)
        # deferred weight gradients: per-layer split-K partials, reduced by the
        # optimizer (mq_grad_src) instead of a reduction launch per layer
        self.dw_parts = [None] * L
        self.dw_nparts = torch.zeros(max(L, 1), dtype=torch.int32, device=dev)
        self.y_nparts = torch.zeros(max(L, 1), dtype=torch.int32, device=dev)
        self._src_key = None
        self._src = None

    def grad_src(self, model: DeviceModel):
        """The _lib.GradSrc describing where each layer's gradient lives this
        step (head partials, deferred tcgen05 partials, or model.flat_g)."""
        key = tuple(int(self.af0 and l == 0 or lib().mq_sage_dw_deferred(self.dims[l + 1]))
                    for l in range(self.L - 1))
        if key == self._src_key and self._src is not None:
            return self._src
        src = GradSrc()
        segs = []
        L = self.L
        seg = GradSrc().seg[0]
        lib().mq_sage_head_grad_seg(self.sw.batch_size, self.dims[L - 1], self.C,
                                    ptr(self.head_scratch), model.offsets[L - 1], C.byref(seg))
        segs.append(seg)
        for l in range(L - 1):
            if l == 0 and self.af0:
                d0, d1 = self.dims[0], self.dims[1]
                if self.dw_parts[0] is None:
                    nb = int(lib().mq_sage_af_dw_parts_bytes(d0, d1))
                    self.dw_parts[0] = torch.zeros(nb // 4 + 1, dtype=torch.float32,
                                                   device=self.sw.graph.device)
                s2 = GradSrc().seg[0]
                s2.part = ptr(self.dw_parts[0])
                s2.nparts_dev = ptr(self.dw_nparts[0:1])
                s2.stride = 2 * d0 * d1
                s2.offset = model.offsets[0]
                s2.size = 2 * d0 * d1
                s2.nparts = 0
                s2.kind = 0
                s2.d_in = d0
                s2.d_out = d1
                segs.append(s2)
            elif key[l]:
                if self.dw_parts[l] is None:
                    nb = int(lib().mq_sage_dw_parts_bytes(self.dims[l], self.dims[l + 1]))
                    self.dw_parts[l] = torch.zeros(nb // 4 + 1, dtype=torch.float32,
                                                   device=self.sw.graph.device)
                s2 = GradSrc().seg[0]
                lib().mq_sage_dw_grad_seg(ptr(self.dw_parts[l]), ptr(self.dw_nparts[l:l + 1]),
                                          self.dims[l], self.dims[l + 1], model.offsets[l],
                                          C.byref(s2))
                segs.append(s2)
        src.nseg = len(segs)
        for i, sg in enumerate(segs):
            src.seg[i] = sg
        self._src_key, self._src = key, src
        return src

    def materialize_grads(self, model: DeviceModel, stream):
        """Resolve the deferred gradient into model.flat_g (tests, eager API)."""
        src = self.grad_src(model)
        tmp = torch.empty_like(model.flat_g)
        lib().mq_grad_reduce(C.byref(src), ptr(model.flat_g), model.num_params, ptr(tmp), stream)
        model.flat_g.copy_(tmp)

    def h_in(self, l, sw):
        return sw.x0 if l == 0 else self.act[l]

    launch_gather = staticmethod(TrainWorkspace.launch_gather)

    def launch_optimizer(self, model: DeviceModel, optimizer: str, stream, grad64=None,
                         scale=1.0):
        TrainWorkspace.launch_optimizer(model, optimizer, stream, grad64=grad64, scale=scale,
                                        src=self.grad_src(model))

    def launch_train(self, model: DeviceModel, stream, sw, ring=None, ring_len=0, world=1):
        """Forward, loss and backward of one batch; gradients land in
        model.flat_g (or its deferred partials, grad_src).  With ``ring`` the
        batch loss is committed to it (mq_step_commit fused into the head);
        otherwise it accumulates in ``self.loss``."""
        for _, op in self.train_ops(model, sw, ring, ring_len, world):
            op(stream)

    def train_ops(self, model: DeviceModel, sw, ring=None, ring_len=0, world=1):
        """The step as an ordered list of (kernel family, fn(stream)) — one C-ABI
        call each, so a profiler can time every launch in isolation."""
        L, d, ld = self.L, self.dims, self.ld_in
        lb = lib()
        self.grad_src(model)  # allocate the deferred partial buffers before capture
        ops = []
        for l in range(L - 1):
            h = L - 1 - l
            hb, b = sw.hops[h], sw.bounds[h]
            if l == 0 and self.af0:
                ops.append(("sage_spmm_l0", lambda s, h=h, hb=hb, b=b:
                            lb.mq_spmm_fwd(ptr(hb.row_ptr), ptr(hb.cols), ptr(hb.vals),
                                           ptr(sw.n_dst_dev(h)), b.n_dst_max, ptr(sw.x0), ld[0],
                                           d[0], ptr(self.agg0), ld[0], s)))
                ops.append(("sage_linear_af_l0", lambda s, h=h, b=b:
                            lb.mq_sage_linear_af(ptr(self.agg0), ld[0], ptr(sw.x0), ld[0],
                                                 ptr(sw.n_dst_dev(h)), b.n_dst_max, d[0],
                                                 ptr(model.weight(0)), d[1], ptr(self.act[1]),
                                                 ld[1], ptr(self.af_part), s)))
                if L == 2:  # the head scatters into dh[1]; TF's aggregation clears it
                    ops.append(("sage_zero_dh", lambda s: lb.mq_memset_async(
                        ptr(self.dh[L - 1]), 0, self.dh[L - 1].numel() * 4, s)))
                continue
            # tensor-core backend: Y stays as split-K partials, summed by the aggregation
            yn = self.y_nparts[l:l + 1] if lb.mq_sage_y_deferred(d[l + 1]) else None
            ops.append((f"sage_transform_l{l}", lambda s, l=l, hb=hb, b=b, yn=yn:
                        lb.mq_sage_transform(ptr(self.h_in(l, sw)), ld[l], ptr(hb.counts),
                                             b.n_src_max, d[l], ptr(model.weight(l)), d[l + 1],
                                             None if yn is not None else ptr(self.Y[l]),
                                             ptr(self.scratch),
                                             ptr(self.Y[l]) if yn is not None else None,
                                             ptr(yn), s)))
            z1 = (self.dh[L - 1], sw.hops[0].counts, ld[L - 1]) if l == L - 2 else (None, None, 0)
            ops.append((f"sage_aggregate_l{l}", lambda s, l=l, h=h, hb=hb, b=b, yn=yn, z1=z1:
                        lb.mq_sage_aggregate(ptr(hb.row_ptr), ptr(hb.cols), ptr(hb.vals),
                                             ptr(sw.n_dst_dev(h)), b.n_dst_max, ptr(self.Y[l]),
                                             d[l + 1], ptr(yn),
                                             ptr(hb.counts) if yn is not None else None,
                                             ptr(self.act[l + 1]), ld[l + 1], ptr(self.G[l]),
                                             ptr(hb.counts), 2 * d[l + 1], ptr(z1[0]),
                                             ptr(z1[1]), z1[2], s)))
        hb0 = sw.hops[0]
        ops.append(("sage_head", lambda s:
                    lb.mq_sage_head(ptr(hb0.row_ptr), ptr(hb0.cols), ptr(hb0.vals),
                                    ptr(sw.n_targets), sw.batch_size, ptr(self.h_in(L - 1, sw)),
                                    ld[L - 1], d[L - 1], ptr(model.weight(L - 1)), self.C,
                                    ptr(sw.labels), None, ptr(self.dh[L - 1]), ld[L - 1],
                                    ptr(self.loss), ptr(sw.key), world, ptr(ring), ring_len,
                                    ptr(model.nonfinite), ptr(self.head_scratch), s)))
        for l in range(L - 2, -1, -1):
            h = L - 1 - l
            hb, b = sw.hops[h], sw.bounds[h]
            if l == 0 and self.af0:
                ops.append(("sage_linear_af_bwd_l0", lambda s, h=h, b=b:
                            lb.mq_sage_linear_af_bwd(ptr(self.agg0), ld[0], ptr(sw.x0), ld[0],
                                                     ptr(sw.n_dst_dev(h)), b.n_dst_max, d[0],
                                                     ptr(self.dh[1]), ld[1], ptr(self.act[1]),
                                                     ld[1], d[1], ptr(self.dw_parts[0]),
                                                     ptr(self.dw_nparts[0:1]), s)))
                continue
            ops.append((f"sage_scatter_bwd_l{l}", lambda s, l=l, h=h, hb=hb, b=b:
                        lb.mq_sage_scatter_bwd(ptr(hb.row_ptr), ptr(hb.cols), ptr(hb.vals),
                                               ptr(sw.n_dst_dev(h)), b.n_dst_max,
                                               ptr(self.dh[l + 1]), ld[l + 1],
                                               ptr(self.act[l + 1]), ld[l + 1], d[l + 1],
                                               ptr(self.G[l]), s)))
            dp = self.dw_parts[l]
            ops.append((f"sage_transform_bwd_l{l}", lambda s, l=l, hb=hb, b=b, dp=dp:
                        lb.mq_sage_transform_bwd(ptr(self.h_in(l, sw)), ld[l], ptr(hb.counts),
                                                 b.n_src_max, d[l], ptr(model.weight(l)),
                                                 d[l + 1], ptr(self.G[l]), ptr(model.grad(l)),
                                                 ptr(self.dh[l]), ld[l], ptr(self.scratch),
                                                 ptr(dp),
                                                 ptr(self.dw_nparts[l:l + 1])
                                                 if dp is not None else None, s)))
        return ops


def current_stream(device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


class capture_graph:
    """torch.cuda.graph with Python's cyclic GC paused: a CUDAGraph of an
    earlier runner collected mid-capture would destroy its graph exec inside
    the capture and invalidate it (cudaErrorStreamCaptureInvalidated)."""

    def __init__(self, graph, stream):
        self._ctx = torch.cuda.graph(graph, stream=stream)

    def __enter__(self):
        import gc
        gc.collect()
        self._was = gc.isenabled()
        gc.disable()
        return self._ctx.__enter__()

    def __exit__(self, *exc):
        import gc
        try:
            return self._ctx.__exit__(*exc)
        finally:
            if self._was:
                gc.enable()
