"""GPU: the production prep pass at BASELINE's full shapes vs the oracle.

One device-planned group of Q = 8 batches x 1024 seeds (setup_q slicing the
epoch permutation, sample_q, the relabel chain, gather_q, labels_q — exactly
what StepRunner / bench.py run) compared slot by slot, array-equal, with
oracle.sampler.build_minibatch: every hop's rows / cols / f64 values /
src_ids / dst_ids, the gathered f32 features and the digest.

* Reddit-shaped (configs[1]): 232,965 nodes, 114M arcs, 602-d, [10,5], 1 %
  degree cache — the headline workload;
* products-shaped (configs[2]): 2.45M nodes, 62M arcs, 100-d, [15,10,5],
  1 % degree cache, plus the host-store miss path (configs[3]).
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu, pytest.mark.slow]
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2601_04707_b200 as mq  # noqa: E402
from paper_2601_04707_b200 import synth  # noqa: E402
from test_gpu_prep import _device_plan_vs_oracle  # noqa: E402


class _Host:
    """Host (oracle-side) view of a device graph."""

    def __init__(self, g):
        self.row_offsets = g.row_off.cpu().numpy()
        self.col_indices = g.col.cpu().numpy()
        self.features = g.features[:, :g.feature_dim].cpu().numpy()
        self.labels = g.labels.cpu().numpy()
        self.train_mask = g.train_mask
        self.num_nodes = g.num_nodes


def _shape(name, placement="hbm", fraction=0.01):
    sg, fanouts = synth.generate_shape(name, seed=0, device="cuda")
    mask = synth.degree_cache_mask(sg.col_indices, sg.num_nodes, fraction).cpu().numpy()
    g = mq.DeviceGraph.from_csr(sg, feature_placement=placement)
    cache = mq.DeviceCache(g, mask, fraction)
    return g, cache, mask, fanouts


def test_reddit_group_vs_oracle():
    g, cache, mask, fanouts = _shape("reddit")
    assert g.feature_dim == 602 and tuple(fanouts) == (10, 5)
    hg = _Host(g)
    _device_plan_vs_oracle(hg, g, cache, mask, fanouts, 1024, seed=0, epoch=0)
    # a later epoch's key and a second group of the same epoch (cursor at Q)
    _device_plan_vs_oracle(hg, g, cache, mask, fanouts, 1024, seed=0, epoch=5, check_slots=3)


@pytest.mark.parametrize("placement", ["hbm", "host"])
def test_products_group_vs_oracle(placement):
    g, cache, mask, fanouts = _shape("products", placement)
    assert tuple(fanouts) == (15, 10, 5)
    hg = _Host(g)
    _device_plan_vs_oracle(hg, g, cache, mask, fanouts, 1024, seed=1, epoch=2,
                           check_slots=8 if placement == "hbm" else 2)


def test_products_fused_step_vs_oracle():
    """The fused training step at the products shape (3 layers, aggregate-
    first 100-d input layer, 1024 seeds, the real prep pass): loss at rel
    1e-5 and per-layer gradients within 1e-5 of the exact (f64) evaluation of
    the same fp32 model on the oracle's identical batch, two windows."""
    from conftest import HostGraph
    from test_gpu_fused import _fused_vs_oracle
    g, _, mask, fanouts = _shape("products")
    h = _Host(g)
    hg = HostGraph(h.row_offsets, h.col_indices, h.features, h.labels, g.num_classes,
                   train_mask=g.train_mask)
    del g
    torch.cuda.empty_cache()
    _fused_vs_oracle(hg, tuple(fanouts), 64, 1024, seed=3, mask=mask, windows=2, layer0="af")


def test_products_group_vs_oracle_hashed_ranks(monkeypatch):
    """The same products-shape group with the relabel's rank words in the
    hashed layout (the one papers-sized graphs use)."""
    monkeypatch.setenv("MQ_PREP_HASH", "1")
    g, cache, mask, fanouts = _shape("products")
    _device_plan_vs_oracle(_Host(g), g, cache, mask, fanouts, 1024, seed=4, epoch=1,
                           check_slots=4)
