"""GPU: the fused SAGE step (csrc/mq_fused.cu) against the CPU oracle.

The StepRunner's default step evaluates hidden layers transform-first and the
last layer as one fused head kernel.  Sampling and gather are
bit-exact, so the oracle (the reference's aggregate-first nn.py restated) sees
the identical batch; loss and gradients agree up to fp32 re-association:
loss rel 1e-5, gradients max|a-b| <= 2e-5 * max|b| per layer.
"""

import os

import numpy as np
import pytest

from conftest import HostGraph, make_cfg1, make_g2

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2601_04707_b200 as mq  # noqa: E402
from oracle import nn as onn  # noqa: E402
from oracle import sampler as osamp  # noqa: E402
from paper_2601_04707_b200.graph import DeviceGraph  # noqa: E402
from paper_2601_04707_b200.runtime import epoch_permutation  # noqa: E402

GRAD_RTOL = 2e-5
EXACT_LOG = []  # (layer, device vs exact, fp32 reference vs exact)


class _Blk64:
    """An oracle block with the forward's float32(1/s) weights held in f64."""

    def __init__(self, b):
        self.rows, self.cols, self.dst_in_src = b.rows, b.cols, b.dst_in_src
        self.values = b.values.astype(np.float32).astype(np.float64)
        self.num_dst, self.num_src = b.num_dst, b.num_src


def _exact_grads(mb, weights, pre32):
    """Gradients of the fp32 model's inputs evaluated in f64 (with the given
    ReLU masks)."""
    layers = [_Blk64(b) for b in mb.layers]
    w64 = [np.asarray(w, np.float64) for w in weights]
    logits, cache = onn.sage_forward(layers, np.asarray(mb.features, np.float64), w64)
    _, dl = onn.batch_loss(logits, mb.target_labels)
    cache["pre"] = [np.asarray(p, np.float64) for p in pre32]
    return onn.backward(layers, w64, cache, dl)


def _normwise(got, ref):
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    return np.abs(got - ref).max() / max(np.abs(ref).max(), 1e-30)


def _fused_vs_oracle(hg, fanouts, hidden, B, seed, mask=None, windows=1, layer0="auto"):
    """Run `windows` eager fused steps on device (compute only, no optimizer)
    and compare loss + gradients of each batch with the oracle."""
    g = DeviceGraph.from_csr(hg)
    cache = mq.DeviceCache(g, mask) if mask is not None else None
    L = len(fanouts)
    C = int(hg.num_classes)
    state = mq.init_model(hg.feature_dim, hidden, C, num_layers=L, seed=7, learning_rate=0.01)
    model = onn.init_model(hg.feature_dim, hidden, C, num_layers=L, seed=7, learning_rate=0.01)
    perm = epoch_permutation(hg.train_mask, seed, 0)
    runner = mq.StepRunner(g, state, fanouts=fanouts, batch_size=B, num_train=perm.size,
                           cache=cache, seed=seed, use_graph=False, pipeline=False,
                           layer0=layer0)
    assert runner.fused
    if layer0 != "auto":
        assert runner.tw.af0 == (layer0 == "af")
    runner.begin_epoch(0, perm)
    if os.environ.get("MQ_TEST_DEFERRED_FIRST"):
        runner.tw.grad_src(state.dev)  # diagnostics: the deferred path from window 0
    s = runner.stream
    for j in range(windows):
        q = j % runner.Q  # one batched prep pass fills Q slots
        sw = runner.groups[0].slots[q]
        with torch.cuda.stream(s):
            if q == 0:
                runner._enqueue_prep(sw, s.cuda_stream)
            runner._enqueue_train(sw, s.cuda_stream, commit=False)
            runner.tw.materialize_grads(state.dev, s.cuda_stream)
        torch.cuda.synchronize()
        loss = float(runner.tw.loss.item())
        runner.tw.loss.zero_()
        assert int(state.dev.nonfinite.item()) == 0
        grads = [state.dev.grad(l).cpu().numpy() for l in range(L)]
        tg = perm[j * B:(j + 1) * B]
        mb = osamp.build_minibatch(hg.row_offsets, hg.col_indices, hg.features, hg.labels, tg,
                                   fanouts, seed=seed, epoch=0, batch_id=j, cached_mask=mask)
        logits, cache = onn.sage_forward(mb.layers, mb.features, model.weights)
        oloss, dlogits = onn.batch_loss(logits, mb.target_labels)
        assert abs(loss - oloss) <= 1e-5 * abs(oloss), (j, loss, oloss)
        # A hidden pre-activation within rounding of 0 may take the other side
        # of the ReLU here than in the oracle (the fused path re-associates the
        # sums).  Back-propagate the oracle through OUR masks so the gradient
        # bar stays rounding-level (the flip itself is legitimate fp32 noise).
        for l in range(L - 1):
            ours = runner.tw.act[l + 1][:cache["pre"][l].shape[0], :cache["pre"][l].shape[1]]
            # (act is shared by all slots and was last written by slot q's step)
            cache["pre"][l] = ours.cpu().numpy()
        ograds = onn.backward(mb.layers, model.weights, cache, dlogits)
        for l, (a, b) in enumerate(zip(grads, ograds)):
            assert a.shape == b.shape
            err = _normwise(a, b)
            assert err <= GRAD_RTOL, (j, l, err)
        # The 2e-5 above compares two fp32 evaluations (ours: 3xTF32 tensor-core
        # contractions with split-K; the reference's: OpenBLAS sgemm), so it
        # carries BOTH rounding errors.  Against the exact arithmetic of the same
        # fp32 inputs (f64 evaluation, float32(1/s) weights, our ReLU masks) the
        # device gradients meet north_star's 1e-5 per layer, and the fp32
        # reference itself is no closer (EXACT_LOG records both).
        g64 = _exact_grads(mb, model.weights, [c for c in cache["pre"]])
        for l, (a, b, c) in enumerate(zip(grads, ograds, g64)):
            e_dev, e_ref = _normwise(a, c), _normwise(b, c)
            EXACT_LOG.append((l, e_dev, e_ref))
            assert e_dev <= 1e-5, (j, l, e_dev, e_ref)


@pytest.fixture(scope="module")
def cfg1():
    return make_cfg1()


LAYER0 = ["tf", "af"]  # input layer transform-first / aggregate-first (engine.py)


@pytest.mark.parametrize("layer0", LAYER0)
def test_fused_two_layer_cfg1(cfg1, layer0):
    _fused_vs_oracle(cfg1, (10, 5), 64, 1024, seed=3, windows=3, layer0=layer0)


@pytest.mark.parametrize("layer0", LAYER0)
def test_fused_two_layer_cfg1_cached(cfg1, layer0):
    rng = np.random.default_rng(0)
    mask = np.zeros(cfg1.num_nodes, bool)
    mask[rng.choice(cfg1.num_nodes, 100, replace=False)] = True
    _fused_vs_oracle(cfg1, (10, 5), 64, 1024, seed=4, mask=mask, windows=2, layer0=layer0)


@pytest.mark.parametrize("layer0", LAYER0)
def test_fused_three_layer_g2(golden_sampling, layer0):
    hg = make_g2(golden_sampling)
    _fused_vs_oracle(hg, (6, 4, 3), 32, 200, seed=5, mask=golden_sampling["g2/mask10"], windows=4,
                     layer0=layer0)


def test_fused_af_products_like_widths():
    """aggregate-first input layer at a products-like width ratio (100-d in,
    64 hidden, 3 layers, big fanouts) on a random graph."""
    rng = np.random.default_rng(21)
    n = 6000
    src = rng.integers(0, n, 120_000)
    dst = (src + rng.integers(1, 2000, src.size)) % n
    keys = np.unique(np.concatenate([src * n + dst, dst * n + src]))
    s, d = keys // n, keys % n
    ro = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(s, minlength=n), out=ro[1:])
    feats = rng.standard_normal((n, 100)).astype(np.float32)
    labels = rng.integers(0, 47, n).astype(np.int32)
    hg = HostGraph(ro, d, feats, labels, 47, rng.random(n) < 0.3)
    _fused_vs_oracle(hg, (15, 10, 5), 64, 512, seed=12, windows=2, layer0="af")


def test_fused_wide_input_layer():
    """Reddit-like input width (602-d, pitch 604, transform-first): the
    swapped tcgen05 weight gradient with X^T tiled over 5 feature tiles and
    deferred split-K partials, against the oracle."""
    rng = np.random.default_rng(31)
    n = 4000
    src = rng.integers(0, n, 60_000)
    dst = (src + rng.integers(1, 500, src.size)) % n
    keys = np.unique(np.concatenate([src * n + dst, dst * n + src]))
    s, d = keys // n, keys % n
    ro = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(s, minlength=n), out=ro[1:])
    feats = rng.standard_normal((n, 602)).astype(np.float32)
    labels = rng.integers(0, 41, n).astype(np.int32)
    hg = HostGraph(ro, d, feats, labels, 41, rng.random(n) < 0.4)
    _fused_vs_oracle(hg, (10, 5), 64, 512, seed=17, windows=2, layer0="tf")


def test_fused_one_layer(golden_sampling):
    hg = make_g2(golden_sampling)
    _fused_vs_oracle(hg, (7,), 16, 128, seed=6, windows=2)


def test_fused_odd_widths():
    """d_in = 30 (pitch 32, pad columns), hidden 13 (odd: scalar paths), 7 classes."""
    rng = np.random.default_rng(11)
    n = 3000
    src = rng.integers(0, n, 40_000)
    dst = (src + rng.integers(1, 200, src.size)) % n
    keys = np.unique(np.concatenate([src * n + dst, dst * n + src]))
    s, d = keys // n, keys % n
    ro = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(s, minlength=n), out=ro[1:])
    feats = rng.standard_normal((n, 30)).astype(np.float32)
    labels = rng.integers(0, 7, n).astype(np.int32)
    train = rng.random(n) < 0.5
    hg = HostGraph(ro, d, feats, labels, 7, train)
    _fused_vs_oracle(hg, (5, 4, 3), 13, 256, seed=9, windows=2)


def test_fused_epoch_matches_unfused(golden_sampling):
    """A whole graph-captured epoch: fused and per-op step agree to training tolerance."""
    hg = make_g2(golden_sampling)
    g = DeviceGraph.from_csr(hg)
    cache = mq.DeviceCache(g, golden_sampling["g2/mask10"])
    out = {}
    for fused in (True, False):
        cfg = mq.PipelineConfig(num_devices=1, batch_size=64,
                                sampler=mq.SamplerParams("sage", (4, 3), num_layers=2),
                                optimizer="adam", seed=5, fused_step=fused)
        st = mq.init_model(16, 16, 5, num_layers=2, seed=5, learning_rate=0.01)
        stats, _ = mq.run_epoch(g, cache, [st], cfg, epoch=0)
        out[fused] = (np.array([stats.losses[b] for b in sorted(stats.losses)]),
                      [w.cpu().numpy() for w in st.weights])
    np.testing.assert_allclose(out[True][0], out[False][0], rtol=1e-4)
    for a, b in zip(out[True][1], out[False][1]):
        assert np.abs(a - b).max() <= 1e-4 * np.abs(b).max()


def test_fused_ffma_backend(cfg1):
    """The fp32 CUDA-core backend of the dense transforms (no deferred partials)."""
    from paper_2601_04707_b200._lib import lib
    old = lib().mq_get_gemm_backend()
    lib().mq_set_gemm_backend(0)
    try:
        _fused_vs_oracle(cfg1, (10, 5), 64, 1024, seed=8, windows=2)
    finally:
        lib().mq_set_gemm_backend(old)


def test_group_graphs_match_window_graphs(golden_sampling):
    """steps(n) (one graph per slot group, prep forked inside) trains like n
    single-window graph launches; the epoch tail runs window by window."""
    hg = make_g2(golden_sampling)
    g = DeviceGraph.from_csr(hg)
    cache = mq.DeviceCache(g, golden_sampling["g2/mask10"])
    perm = epoch_permutation(hg.train_mask, 5, 0)
    B = 64
    n_win = -(-perm.size // B)
    outs = []
    for grouped in (False, True):
        st = mq.init_model(16, 16, 5, num_layers=2, seed=5, learning_rate=0.01)
        r = mq.StepRunner(g, st, fanouts=(4, 3), batch_size=B, num_train=perm.size, cache=cache,
                          seed=5, queue_depth=3)
        r.begin_epoch(0, perm)
        r.capture()
        if grouped:
            assert r.steps(n_win) == n_win
        else:
            for _ in range(n_win):
                r.step()
        r.check_finite()
        outs.append((r.losses(n_win), [w.cpu().numpy() for w in st.weights]))
    np.testing.assert_allclose(outs[1][0], outs[0][0], rtol=1e-5)
    for a, b in zip(outs[1][1], outs[0][1]):
        assert np.abs(a - b).max() <= 1e-5 * np.abs(b).max()


@pytest.mark.gpu
def test_epoch_boundary_overlap_matches_serial(golden_sampling):
    """steps() across epochs: each epoch's last group runs train-only and the
    next epoch's first prep runs beside it in the other slot group (g0
    alternates).  Losses of every epoch and the final weights match the
    per-window schedule whose epoch boundaries are fully serialised."""
    hg = make_g2(golden_sampling)
    g = DeviceGraph.from_csr(hg)
    cache = mq.DeviceCache(g, golden_sampling["g2/mask10"])
    B, E = 64, 4
    perms = [epoch_permutation(hg.train_mask, 5, e) for e in range(E)]
    n_win = -(-perms[0].size // B)
    outs = []
    for overlapped in (False, True):
        st = mq.init_model(16, 16, 5, num_layers=2, seed=5, learning_rate=0.01)
        r = mq.StepRunner(g, st, fanouts=(4, 3), batch_size=B, num_train=perms[0].size,
                          cache=cache, seed=5, queue_depth=3)
        r.begin_epoch(0, perms[0])
        r.capture()
        c_last = (n_win - 1) % 3 + 1
        assert f"tgroup0_{c_last}" in r.graphs and f"tgroup1_{c_last}" in r.graphs
        losses, starts = [], []
        for e in range(E):
            if e:
                r.begin_epoch(e, perms[e])
            starts.append(r.g0)
            if overlapped:
                assert r.steps(n_win) == n_win
                assert r._tail_clean
            else:
                for _ in range(n_win):
                    r.step()
            # the epoch's losses copied on the train stream: no host sync, so
            # the next begin_epoch really overlaps this epoch's last group
            with torch.cuda.stream(r.stream):
                losses.append(r.loss_ring[:n_win].clone())
        r.check_finite()
        losses = [x.cpu().numpy() for x in losses]
        if overlapped and -(-n_win // 3) % 2 == 1:  # odd group count: the start group alternates
            assert starts == [0, 1, 0, 1]
        outs.append((losses, [w.cpu().numpy() for w in st.weights]))
    for a, b in zip(outs[1][0], outs[0][0]):
        np.testing.assert_allclose(a, b, rtol=1e-5)
    for a, b in zip(outs[1][1], outs[0][1]):
        assert np.abs(a - b).max() <= 1e-5 * np.abs(b).max()


@pytest.mark.gpu
def test_steps_tails_defer_the_next_prep(golden_sampling):
    """steps() calls that end inside a slot group run the tail train-only and
    hold the next group's prep back until the next call (_flush_prep); calls
    of 5 and 4 windows mix group graphs, deferred tails and single windows and
    still train like one window at a time."""
    hg = make_g2(golden_sampling)
    g = DeviceGraph.from_csr(hg)
    cache = mq.DeviceCache(g, golden_sampling["g2/mask10"])
    perm = epoch_permutation(hg.train_mask, 5, 0)
    B = 64
    n_win = -(-perm.size // B)
    outs = []
    for chunked in (False, True):
        st = mq.init_model(16, 16, 5, num_layers=2, seed=5, learning_rate=0.01)
        r = mq.StepRunner(g, st, fanouts=(4, 3), batch_size=B, num_train=perm.size, cache=cache,
                          seed=5, queue_depth=3)
        r.begin_epoch(0, perm)
        r.capture()
        done, deferred = 0, 0
        while done < n_win:
            if chunked:
                done += r.steps(5 if (done // 5) % 2 == 0 else 4)
                deferred += r._pending_prep is not None
            else:
                r.step()
                done += 1
        if chunked:
            assert deferred > 0
        r.check_finite()
        outs.append((r.losses(n_win), [w.cpu().numpy() for w in st.weights]))
    np.testing.assert_allclose(outs[1][0], outs[0][0], rtol=1e-5)
    for a, b in zip(outs[1][1], outs[0][1]):
        assert np.abs(a - b).max() <= 1e-5 * np.abs(b).max()
