"""GPU: run_epoch's Trace and queue statistics come from device stage stamps.

The reference emits a span around every stage of every batch
(runtime.py:399-401, 444-447, 478-481, 533-546; schema pipeline.py:24-98)
and logs queue high-water marks and put/get key orders (pipeline.py:109-167,
checked for conservation and FIFO order in test_runtime.py:197-208).  Here
the spans are read from GPU-clock stamps recorded in the step graphs, so the
trace shows the real overlap of the prep stream (sample, transfer) with the
train stream (compute, share, apply).
"""

import numpy as np
import pytest

from conftest import make_g2

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2601_04707_b200 as mq  # noqa: E402


def _run(golden_sampling, golden_runtime, G, trace=True, epochs=1):
    hg = make_g2(golden_sampling)
    hg.train_mask = golden_runtime["epoch/train_mask"]
    g = mq.DeviceGraph.from_csr(hg)
    cache = mq.DeviceCache(g, golden_sampling["g2/mask10"])
    cfg = mq.PipelineConfig(num_devices=G, batch_size=32, queue_capacity=4,
                            sampler=mq.SamplerParams("sage", (4, 3), num_layers=2),
                            optimizer="adam", sync_period=2, seed=5, trace=trace)
    base = mq.init_model(16, 16, 5, num_layers=2, seed=5, learning_rate=0.01)
    reps = [base.copy() for _ in range(G)]
    tr = mq.Trace()
    stats = []
    for e in range(epochs):
        st, _ = mq.run_epoch(g, cache, reps, cfg, epoch=e, trace=tr)
        stats.append(st)
    return stats, tr, cfg


@pytest.mark.parametrize("G", [1, 2])
def test_stage_spans_from_device_stamps(golden_sampling, golden_runtime, G):
    stats, tr, cfg = _run(golden_sampling, golden_runtime, G, epochs=2)
    for e, st in enumerate(stats):
        for d in range(G):
            per_dev = st.queue_keys[d]["dev_get"]
            assert per_dev, "device got no batches"
            # FIFO and conservation (test_runtime.py:197-208)
            assert st.queue_keys[d]["dev_put"] == per_dev == st.queue_keys[d]["cpu_put"]
            assert sorted(per_dev) == sorted(b for b in st.losses if b % G == d)
            hw = st.queue_high_water[d]
            assert 1 <= hw["dev"] <= 2 * cfg.queue_capacity and hw["cpu"] >= 1
            evs = {}
            for ev in tr.events(device=d):
                if ev.epoch == e:
                    evs.setdefault((ev.stage, ev.batch), []).append(ev)
            for bid in per_dev:
                one = {s: evs[(s, bid)][0] for s in ("sample", "transfer", "enqueue_dev",
                                                     "compute_fwd", "compute_bwd", "grad_share")}
                assert one["sample"].t_end_ns <= one["transfer"].t_start_ns + 0
                assert one["transfer"].t_end_ns <= one["compute_fwd"].t_start_ns
                assert one["enqueue_dev"].t_start_ns == one["transfer"].t_end_ns
                assert one["enqueue_dev"].t_end_ns == one["compute_fwd"].t_start_ns
                assert one["compute_fwd"].t_end_ns == one["compute_bwd"].t_start_ns
                assert one["compute_bwd"].t_end_ns <= one["grad_share"].t_end_ns
                assert one["compute_fwd"].t_end_ns > one["compute_fwd"].t_start_ns
            applies = [ev for ev in tr.events(stage="grad_apply", device=d) if ev.epoch == e]
            assert len(applies) == -(-len(st.losses) // G)  # every window, on every device
            syncs = [ev for ev in tr.events(stage="sync", device=d) if ev.epoch == e]
            assert len(syncs) == st.sync_count + st.epoch_sync
        # compute busy fraction of the traced span, measured on the GPU clock
        u = mq.utilization(tr, device=0)
        assert 0.0 < u <= 1.0


def test_stamps_do_not_change_results(golden_sampling, golden_runtime):
    a, _, _ = _run(golden_sampling, golden_runtime, 1, trace=True)
    b, _, _ = _run(golden_sampling, golden_runtime, 1, trace=False)
    bids = sorted(a[0].losses)
    np.testing.assert_allclose([a[0].losses[k] for k in bids], [b[0].losses[k] for k in bids],
                               rtol=1e-6)
