"""CPU restatement of the SAGE numerics — test oracle.

Follows ``mqpipe/nn.py`` of the reference:

* ``init_model``   — ``nn.py:56-71`` (Glorot uniform, SAGE fan-in doubled)
* ``block_apply``  — ``nn.py:79-89`` (``np.add.at`` row-ordered segment sum)
* ``block_apply_t``— ``nn.py:92-98``
* ``sage_forward`` — ``nn.py:116-133``
* ``batch_loss``   — ``nn.py:141-156`` (summed softmax-CE)
* ``backward``     — ``nn.py:159-180`` (SAGE arm)
* ``adam_step``    — ``nn.py:191-206`` (beta 0.9/0.999, eps 1e-8; NumPy-2
  weak-scalar f32 arithmetic)
* ``sgd_step``     — ``nn.py:209-215``
* ``full_forward`` — ``nn.py:218-250`` (sage arm), ``accuracy`` — ``nn.py:253-256``

Blocks are any objects with ``rows, cols, values, num_dst, dst_in_src``.
"""

from __future__ import annotations

import numpy as np

ADAM_BETA1 = 0.9
ADAM_BETA2 = 0.999
ADAM_EPS = 1e-8


class OracleModel:
    def __init__(self, weights, learning_rate=0.001):
        self.weights = weights
        self.learning_rate = learning_rate
        self.step_count = 0
        self.m = [np.zeros_like(w) for w in weights]
        self.v = [np.zeros_like(w) for w in weights]

    def copy(self):
        o = OracleModel([w.copy() for w in self.weights], self.learning_rate)
        o.step_count = self.step_count
        o.m = [m.copy() for m in self.m]
        o.v = [v.copy() for v in self.v]
        return o


def glorot_weights(dims, seed, dtype=np.float32):
    """SAGE weights (2*d_l, d_{l+1}) drawn as in nn.py:56-71."""
    rng = np.random.default_rng(seed)
    out = []
    for l in range(len(dims) - 1):
        fan_in, fan_out = 2 * dims[l], dims[l + 1]
        limit = np.sqrt(6.0 / (fan_in + fan_out))
        out.append(rng.uniform(-limit, limit, size=(fan_in, fan_out)).astype(dtype))
    return out


def init_model(feature_dim, hidden_dim, num_classes, num_layers=2, seed=0,
               learning_rate=0.001, dtype=np.float32):
    dims = [feature_dim] + [hidden_dim] * (num_layers - 1) + [num_classes]
    return OracleModel(glorot_weights(dims, seed, dtype), learning_rate)


def block_apply(blk, h):
    out = np.zeros((blk.num_dst, h.shape[1]), dtype=h.dtype)
    if blk.rows.size:
        vals = blk.values.astype(h.dtype)
        np.add.at(out, blk.rows, vals[:, None] * h[blk.cols])
    return out


def block_apply_t(blk, grad, num_src):
    out = np.zeros((num_src, grad.shape[1]), dtype=grad.dtype)
    if blk.rows.size:
        vals = blk.values.astype(grad.dtype)
        np.add.at(out, blk.cols, vals[:, None] * grad[blk.rows])
    return out


def _check_finite(name, arr):
    if not np.all(np.isfinite(arr)):
        raise FloatingPointError(f"{name} contains NaN or Inf")


def sage_forward(layers, features, weights):
    """Returns (logits, cache) with cache = {'inputs': [(h, both)], 'pre': [z]}."""
    h = np.asarray(features, dtype=weights[0].dtype)
    cache = {"inputs": [], "pre": []}
    last = len(layers) - 1
    for l, blk in enumerate(layers):
        agg = block_apply(blk, h)
        both = np.concatenate([agg, h[blk.dst_in_src]], axis=1)
        cache["inputs"].append((h, both))
        z = both @ weights[l]
        cache["pre"].append(z)
        h = np.maximum(z, 0) if l < last else z
    _check_finite("sage_forward output", h)
    return h, cache


def batch_loss(logits, labels):
    labels = np.asarray(labels)
    shifted = logits - logits.max(axis=1, keepdims=True)
    exp = np.exp(shifted)
    denom = exp.sum(axis=1, keepdims=True)
    log_probs = shifted - np.log(denom)
    n = logits.shape[0]
    loss = -log_probs[np.arange(n), labels].sum()
    grad = exp / denom
    grad[np.arange(n), labels] -= 1.0
    _check_finite("batch_loss", grad)
    return float(loss), grad


def backward(layers, weights, cache, dlogits):
    grads = [None] * len(weights)
    dz = dlogits.astype(weights[0].dtype)
    for l in range(len(layers) - 1, -1, -1):
        blk = layers[l]
        h_in, both = cache["inputs"][l]
        if l < len(layers) - 1:
            dz = dz * (cache["pre"][l] > 0)
        grads[l] = both.T @ dz
        if l > 0:
            dt = dz @ weights[l].T
            d_in = h_in.shape[1]
            dh = block_apply_t(blk, dt[:, :d_in], h_in.shape[0])
            np.add.at(dh, blk.dst_in_src, dt[:, d_in:])
            dz = dh
    for g in grads:
        _check_finite("backward", g)
    return grads


def loss_and_grads(layers, features, labels, weights):
    logits, cache = sage_forward(layers, features, weights)
    loss, dlogits = batch_loss(logits, labels)
    grads = backward(layers, weights, cache, dlogits)
    return loss, grads, logits


def adam_step(model, grads):
    """In place; f32 arrays with Python-float (weak) scalars, as nn.py:191-206."""
    model.step_count += 1
    t = model.step_count
    lr = model.learning_rate
    for w, g, m, v in zip(model.weights, grads, model.m, model.v):
        g = g.astype(w.dtype)
        m *= ADAM_BETA1
        m += (1 - ADAM_BETA1) * g
        v *= ADAM_BETA2
        v += (1 - ADAM_BETA2) * g * g
        m_hat = m / (1 - ADAM_BETA1 ** t)
        v_hat = v / (1 - ADAM_BETA2 ** t)
        w -= lr * m_hat / (np.sqrt(v_hat) + ADAM_EPS)
        _check_finite("adam_step", w)
    return model


def sgd_step(model, grads):
    model.step_count += 1
    for w, g in zip(model.weights, grads):
        w -= model.learning_rate * g.astype(w.dtype)
        _check_finite("sgd_step", w)
    return model


def full_forward(row_offsets, col_indices, features, weights):
    """Whole-graph SAGE forward (nn.py:218-250, sage arm): mean over the
    out-neighbours with stored self loops dropped (nn.py:236-238), concat the
    node's own embedding, ReLU except after the last layer."""
    n = row_offsets.size - 1
    h = features.astype(np.float32)
    last = len(weights) - 1
    src_all = np.repeat(np.arange(n), np.diff(row_offsets))
    keep = col_indices != src_all
    src, dst = src_all[keep], col_indices[keep]
    counts = np.bincount(src, minlength=n).astype(np.float32)
    inv = np.where(counts > 0, 1.0 / np.maximum(counts, 1), 0.0)
    for l, w in enumerate(weights):
        agg = np.zeros_like(h)
        np.add.at(agg, src, h[dst])
        agg *= inv[:, None]
        z = np.concatenate([agg, h], axis=1) @ w
        h = np.maximum(z, 0) if l < last else z
    _check_finite("full_forward", h)
    return h


def accuracy(logits, labels):
    """nn.py:253-256 (first-max argmax)."""
    if logits.shape[0] == 0:
        return 0.0
    return float((logits.argmax(axis=1) == np.asarray(labels)).mean())
