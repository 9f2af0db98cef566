"""GPU: BASELINE configs[1] at full size (Reddit-shaped, 114M arcs, 602-d).

The oracle is too slow for whole epochs at this size, so parity here is
(1) bit-exact hop-0 blocks against the oracle for a full batch of 1024 seeds,
(2) size-independent invariants of the two-hop blocks (CSR membership,
fanout counts, the GNS hot-preference rule, relabel order), and
(3) the captured training step making progress with finite losses.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu, pytest.mark.slow]
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2601_04707_b200 as mq  # noqa: E402
from oracle import sampler as osamp  # noqa: E402
from paper_2601_04707_b200 import synth  # noqa: E402


@pytest.fixture(scope="module")
def reddit():
    sg, fanouts = synth.generate_shape("reddit", seed=0, device="cuda")
    mask = synth.degree_cache_mask(sg.col_indices, sg.num_nodes, 0.01).cpu().numpy()
    g = mq.DeviceGraph.from_csr(sg)
    cache = mq.DeviceCache(g, mask, 0.01)
    ro = g.row_off.cpu().numpy()
    col = g.col.cpu().numpy()
    return sg, g, cache, mask, ro, col, fanouts


def test_shape(reddit):
    sg, g, cache, mask, ro, col, fanouts = reddit
    assert g.num_nodes == 232_965 and g.feature_dim == 602 and g.num_classes == 41
    assert 114_000_000 <= g.num_edges <= 114_200_000
    assert g.self_loops == 0
    assert cache.size == int(np.ceil(0.01 * g.num_nodes))
    # residency index == hot arcs
    assert cache.num_hot_arcs == int(mask[col].sum())


def test_hop0_bit_exact_vs_oracle_full_batch(reddit):
    sg, g, cache, mask, ro, col, fanouts = reddit
    rng = np.random.default_rng(1)
    tg = rng.choice(np.flatnonzero(g.train_mask), size=1024, replace=False)
    blk = mq.node_wise_block(g, tg, 10, mq.PhiloxStream(0, 0, 7, 0), arch="sage", cached_mask=cache)
    ref = osamp.node_wise_block(ro, col, tg, 10, seed=0, epoch=0, batch_id=7, hop=0,
                                cached_mask=mask)
    r = blk.to_reference()
    for k in ("rows", "cols", "values", "src_ids"):
        assert np.array_equal(r[k], getattr(ref, k)), k


def test_two_hop_block_invariants(reddit):
    sg, g, cache, mask, ro, col, fanouts = reddit
    tg = np.flatnonzero(g.train_mask)[:1024]
    mb = mq.build_minibatch(g, tg, mq.SamplerParams("sage", fanouts, 2), mq.PhiloxStream(0, 0, 3),
                            cached_mask=cache)
    deg = np.diff(ro)
    for hop, blk in enumerate(reversed(mb.layers)):
        f = fanouts[hop]
        r = blk.to_reference()
        rows, cols, src, dst = r["rows"], r["cols"], r["src_ids"], r["dst_ids"]
        assert np.all(np.diff(rows) >= 0) and (cols.max() < src.size)
        assert np.array_equal(src[:dst.size], dst)
        assert np.unique(src).size == src.size
        cnt = np.bincount(rows, minlength=dst.size)
        assert np.array_equal(cnt, np.minimum(deg[dst], f))
        assert np.allclose(r["values"], 1.0 / cnt[rows])
        nb = src[cols]
        v = dst[rows]
        # every pick is a real (non-loop) neighbour: binary search in the sorted row
        pos = np.array([np.searchsorted(col[ro[a]:ro[a + 1]], b) for a, b in
                        zip(v[:20000], nb[:20000])])
        assert np.all(col[ro[v[:20000]] + pos] == nb[:20000])
        # GNS rule: a row with >= f resident neighbours samples only residents;
        # otherwise all its residents are sampled
        cs = np.concatenate([[0], np.cumsum(mask[col].astype(np.int64))])
        hot_cnt = cs[ro[dst + 1]] - cs[ro[dst]]
        picked_hot = np.bincount(rows, weights=mask[nb], minlength=dst.size)
        big = deg[dst] > f
        assert np.all(picked_hot[big] == np.minimum(hot_cnt[big], f))
        # first-occurrence relabel: new ids appear in edge order
        new = cols >= dst.size
        firsts = np.unique(cols[new], return_index=True)[1]
        assert np.all(np.diff(cols[new][np.sort(firsts)]) == 1)


def test_captured_training_progresses(reddit):
    sg, g, cache, mask, ro, col, fanouts = reddit
    state = mq.init_model(602, 64, 41, num_layers=2, seed=0, learning_rate=1e-3)
    n_train = int(g.train_mask.sum())
    runner = mq.StepRunner(g, state, fanouts=fanouts, batch_size=1024, num_train=n_train,
                           cache=cache, seed=0)
    runner.begin_epoch(0, mq.runtime.epoch_permutation(g.train_mask, 0, 0))
    runner.capture()
    for _ in range(120):
        runner.step()
    runner.check_finite()
    losses = runner.losses(120) / 1024.0
    assert np.all(np.isfinite(losses))
    assert losses[-20:].mean() < 0.95 * losses[:5].mean()
    assert int(cache.hit_miss.sum()) > 0
