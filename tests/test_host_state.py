"""Host-side optimizer state rules (CPU): the Adam bias-correction table is
allocated once, reaches the saturated (1.0f, 1.0f) row, and is never
replaced (captured graphs hold its pointer; mqgnn.h mq_adam)."""

import numpy as np
import torch

from paper_2601_04707_b200.engine import BIAS_SATURATED, DeviceModel, _bias_table


def test_bias_table_saturates_and_matches_python_floats():
    tab, n = _bias_table(BIAS_SATURATED, "cpu")
    tab = tab.numpy().reshape(-1, 2)
    assert n == BIAS_SATURATED and (tab[-1] == 1.0).all()
    for t in (1, 2, 10, 1000, 17_000, 17_500, BIAS_SATURATED):
        assert tab[t - 1, 0] == np.float32(1 - 0.9 ** t)
        assert tab[t - 1, 1] == np.float32(1 - 0.999 ** t)
    # every t past the table rounds to the last row exactly
    for t in (BIAS_SATURATED + 1, 10 ** 6, 2 ** 31 - 1):
        assert np.float32(1 - 0.9 ** t) == 1.0 and np.float32(1 - 0.999 ** t) == 1.0


def test_bias_table_never_reallocated_and_lr_scalar():
    w = [np.ones((4, 3), np.float32)]
    dm = DeviceModel(w, 1e-3, torch.device("cpu"))
    p = dm.bias.data_ptr()
    dm.ensure_bias(10 ** 7)
    assert dm.bias.data_ptr() == p
    assert float(dm.lr_dev[0]) == np.float32(1e-3)
    dm.learning_rate = 0.25
    assert dm.learning_rate == 0.25 and float(dm.lr_dev[0]) == 0.25
