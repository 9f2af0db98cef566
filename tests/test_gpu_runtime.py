"""GPU: whole-epoch parity of the captured-graph runtime against the reference.

The golden epochs were produced by the reference's own ``run_epoch``
(deterministic serial schedule, 1-3 simulated devices, Adam/SGD, sync period
1-3, with and without a GNS cache).  Sampling and cache statistics must match
exactly; losses and weights within fp32 training tolerance.
"""

import numpy as np
import pytest

from conftest import make_g2

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2601_04707_b200 as mq  # noqa: E402
from paper_2601_04707_b200.graph import DeviceGraph  # noqa: E402


@pytest.fixture(scope="module")
def g2_epoch(golden_sampling, golden_runtime):
    hg = make_g2(golden_sampling)
    hg.train_mask = golden_runtime["epoch/train_mask"]
    return DeviceGraph.from_csr(hg)


CASES = {"1dev_adam": (1, "adam", 1, None), "2dev_adam": (2, "adam", 1, "g2/mask10"),
         "2dev_sgd_p3": (2, "sgd", 3, None), "3dev_adam_p2": (3, "adam", 2, "g2/mask1")}


@pytest.mark.parametrize("name", list(CASES))
@pytest.mark.parametrize("use_graph", [True, False])
def test_run_epoch_matches_reference(golden_runtime, golden_sampling, g2_epoch, name, use_graph):
    rt = golden_runtime
    G, opt, P, mask_name = CASES[name]
    cache = mq.DeviceCache(g2_epoch, golden_sampling[mask_name]) if mask_name else None
    cfg = mq.PipelineConfig(num_devices=G, batch_size=64,
                            sampler=mq.SamplerParams("sage", (4, 3), num_layers=2),
                            optimizer=opt, sync_period=P, seed=5, use_graph=use_graph)
    base = mq.init_model(16, 16, 5, num_layers=2, seed=5, learning_rate=0.01)
    reps = [base.copy() for _ in range(G)]
    stats, trace = mq.run_epoch(g2_epoch, cache, reps, cfg, epoch=1)
    bids = rt[f"epoch/{name}/loss_bids"].tolist()
    assert sorted(stats.losses) == bids
    got = np.array([stats.losses[b] for b in bids])
    np.testing.assert_allclose(got, rt[f"epoch/{name}/losses"], rtol=1e-4)
    assert [stats.sync_count, stats.epoch_sync] == rt[f"epoch/{name}/sync_count"].tolist()
    assert [stats.cache_hits, stats.cache_misses] == rt[f"epoch/{name}/hits"].tolist()
    for l in range(2):
        w = rt[f"epoch/{name}/w{l}"]
        err = np.abs(reps[0].weights[l].cpu().numpy() - w).max()
        assert err <= 1e-4 * np.abs(w).max(), (l, err)
    # every replica ends identical after the epoch barrier (test_runtime.py:174-186)
    for r in reps[1:]:
        for a, b in zip(r.weights, reps[0].weights):
            assert torch.equal(a, b)
    assert len(trace.events(stage="sync")) == G * (stats.sync_count + stats.epoch_sync)


def test_capture_weights_trace(golden_runtime, g2_epoch):
    cfg = mq.PipelineConfig(num_devices=2, batch_size=64,
                            sampler=mq.SamplerParams("sage", (4, 3), num_layers=2),
                            optimizer="sgd", sync_period=3, seed=5, capture_weights=True)
    base = mq.init_model(16, 16, 5, num_layers=2, seed=5, learning_rate=0.01)
    reps = [base.copy() for _ in range(2)]
    stats, _ = mq.run_epoch(g2_epoch, None, reps, cfg, epoch=1)
    wt = stats.weight_traces[0]
    assert [k for k, _ in wt] == golden_runtime["epoch/2dev_sgd_p3/trace_windows"].tolist()
    np.testing.assert_allclose(wt[0][1][0], golden_runtime["epoch/2dev_sgd_p3/trace_w0_first"],
                               rtol=1e-5, atol=1e-7)


def test_host_input_step_matches_graph_step(g2_epoch):
    """The e2e entry point (H2D targets -> graph -> D2H loss) trains the same."""
    fan, B = (4, 3), 64
    perm = mq.runtime.epoch_permutation(g2_epoch.train_mask, 5, 0)
    base = mq.init_model(16, 16, 5, num_layers=2, seed=5, learning_rate=0.01)
    a, b = base.copy(), base.copy()
    ra = mq.StepRunner(g2_epoch, a, fanouts=fan, batch_size=B, num_train=perm.size, seed=5)
    rb = mq.StepRunner(g2_epoch, b, fanouts=fan, batch_size=B, num_train=perm.size, seed=5)
    ra.begin_epoch(0, perm)
    rb.begin_epoch(0, perm)
    ra.capture()
    rb.capture_host_input()
    losses_b = []
    for k in range(5):
        ra.step()
        t = torch.as_tensor(perm[k * B:(k + 1) * B].astype(np.int32)).pin_memory()
        losses_b.append(rb.step_from_host(t, k))
    la = ra.losses(5)
    np.testing.assert_allclose(np.array(losses_b), la, rtol=1e-5)
    for x, y in zip(a.weights, b.weights):
        np.testing.assert_allclose(x.cpu().numpy(), y.cpu().numpy(), rtol=1e-4, atol=1e-6)
