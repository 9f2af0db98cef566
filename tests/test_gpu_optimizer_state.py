"""Optimizer state across long runs and learning-rate changes (GPU).

* Adam past the bias-correction table: steps t > 65,536 read the table's last
  row, which is exactly float32(1 - beta**t) == 1.0f there, so the update
  stays bit-identical to the oracle's adam_step (nn.py:191-206) at any t.
* The table is allocated once (captured graphs hold its pointer).
* Captured step graphs follow ModelState.learning_rate (the kernels read a
  device scalar), as the reference reads state.learning_rate every step.
"""

import numpy as np
import pytest
import torch

from conftest import load_golden, make_g2

pytestmark = pytest.mark.gpu

mq = pytest.importorskip("paper_2601_04707_b200")
from oracle import nn as onn  # noqa: E402


@pytest.mark.parametrize("t0", [17_000, 65_535, 70_000, 1_000_000])
def test_adam_bit_exact_at_large_step_counts(t0):
    gn = load_golden("nn.npz")
    w0 = onn.init_model(16, 32, 5, num_layers=2, seed=7, learning_rate=0.01)
    state = mq.ModelState([w.copy() for w in w0.weights], learning_rate=0.01,
                          step_count=t0, device="cuda")
    ptr_before = state.dev.bias.data_ptr()
    w0.step_count = t0
    for step in range(3):
        grads = [gn[f"2l/s{step}/grad{l}"] for l in range(2)]
        mq.adam_step(state, [torch.as_tensor(g).cuda() for g in grads])
        onn.adam_step(w0, grads)
        for l in range(2):
            assert np.array_equal(state.weights[l].cpu().numpy(), w0.weights[l]), (t0, step, l)
            assert np.array_equal(state.m[l].cpu().numpy(), w0.m[l])
            assert np.array_equal(state.v[l].cpu().numpy(), w0.v[l])
    assert state.step_count == t0 + 3
    assert state.dev.bias.data_ptr() == ptr_before


def test_captured_steps_follow_learning_rate():
    gs = load_golden("sampling.npz")
    hg = make_g2(gs)
    g = mq.DeviceGraph.from_csr(hg, device="cuda:0")
    state = mq.init_model(16, 32, 5, num_layers=2, seed=7, learning_rate=0.0, device="cuda:0")
    runner = mq.StepRunner(g, state, fanouts=(10, 5), batch_size=64,
                           num_train=int(hg.train_mask.sum()), seed=4)
    runner.begin_epoch(0, mq.runtime.epoch_permutation(hg.train_mask, 4, 0))
    runner.capture()
    w_start = [w.cpu().numpy().copy() for w in state.weights]
    for _ in range(2):
        runner.step()
    runner.check_finite()
    for a, b in zip(state.weights, w_start):  # lr 0: Adam moves nothing
        assert np.array_equal(a.cpu().numpy(), b)
    state.learning_rate = 1e-2
    runner.step()
    runner.check_finite()
    moved = [not np.array_equal(a.cpu().numpy(), b) for a, b in zip(state.weights, w_start)]
    assert all(moved)
    state.learning_rate = 0.0
    w_mid = [w.cpu().numpy().copy() for w in state.weights]
    runner.step()
    runner.check_finite()
    for a, b in zip(state.weights, w_mid):
        assert np.array_equal(a.cpu().numpy(), b)
