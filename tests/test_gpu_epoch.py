"""GPU parity of the per-epoch functions around the hot path: full-graph
evaluation (nn.full_forward / evaluate, mq_eval.cu) against the reference-made
fixtures and the oracle.  Bars: logits normwise rel 1e-5
(GEMM re-association), accuracy within 0.5 points (north_star), and
bit-identical results run to run."""

import numpy as np
import pytest

from conftest import epoch_graph, load_golden

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2601_04707_b200 as mq  # noqa: E402
from oracle import nn as onn  # noqa: E402
from paper_2601_04707_b200 import nn as mnn  # noqa: E402

G = load_golden("epoch.npz")
EVAL = sorted({k.split("/")[1] for k in G if k.startswith("eval/")})


def close_normwise(got, ref, rtol=1e-5):
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    assert got.shape == ref.shape
    scale = max(np.abs(ref).max(initial=0.0), 1e-30)
    err = np.abs(got - ref).max(initial=0.0)
    assert err <= rtol * scale, f"max err {err:.3e} vs scale {scale:.3e}"


@pytest.mark.parametrize("tag", EVAL)
@pytest.mark.parametrize("phase", [0, 1])
def test_full_forward_matches_reference(tag, phase):
    g = epoch_graph(G, str(G[f"eval/{tag}/graph"]))
    dg = mq.DeviceGraph.from_csr(g, device="cuda:0")
    p = f"eval/{tag}/p{phase}"
    ws = [G[f"{p}/w{l}"] for l in range(3) if f"{p}/w{l}" in G]
    state = mq.ModelState(ws, device="cuda:0")
    logits = mnn.full_forward(dg, state)
    close_normwise(logits.cpu().numpy(), G[f"{p}/logits"])
    again = mnn.full_forward(dg, state).cpu().numpy()
    assert np.array_equal(again, logits.cpu().numpy())  # deterministic
    for mask, key in ((g.val_mask, "val_acc"), (g.test_mask, "test_acc")):
        acc = mnn.evaluate(dg, state, mask)
        assert abs(acc - float(G[f"{p}/{key}"][0])) <= 0.005 + 1e-12, (key, acc)


def _hub_graph(n=6000, hub_deg=5000, seed=3):
    """Rows that span several 1024-arc work items, isolated rows, self loops."""
    from conftest import HostGraph, csr_from_edges
    rng = np.random.default_rng(seed)
    e = [np.stack([np.zeros(hub_deg, np.int64), rng.choice(np.arange(1, n), hub_deg, replace=False)], 1),
         np.stack([np.full(2500, 7), rng.choice(n, 2500, replace=False)], 1),
         rng.integers(0, n - 100, size=(30000, 2))]
    e = np.concatenate(e)
    e = np.concatenate([e, e[:, ::-1]])
    ro, col = csr_from_edges(e, n)  # nodes >= n-100 with no drawn arc stay isolated
    feats = rng.standard_normal((n, 19)).astype(np.float32)
    labels = rng.integers(0, 7, n).astype(np.int32)
    g = HostGraph(ro, col, feats, labels, 7)
    g.val_mask = rng.random(n) < 0.3
    return g


def test_full_forward_hubs_isolated_and_loops():
    g = _hub_graph()
    assert (np.diff(g.row_offsets) == 0).any()
    dg = mq.DeviceGraph.from_csr(g, device="cuda:0")
    for layers, hidden in ((2, 64), (3, 40)):
        state = mq.init_model(19, hidden, 7, num_layers=layers, seed=2, device="cuda:0")
        ws = [w.cpu().numpy() for w in state.weights]
        ref = onn.full_forward(g.row_offsets, g.col_indices, g.features, ws)
        got = mnn.full_forward(dg, state).cpu().numpy()
        close_normwise(got, ref)
        idx = np.flatnonzero(g.val_mask)
        assert abs(mnn.evaluate(dg, state, g.val_mask) -
                   onn.accuracy(ref[idx], g.labels[idx])) <= 0.005


@pytest.mark.parametrize("tag", EVAL)
def test_lean_evaluate_matches_reference(tag, monkeypatch):
    """the memory-lean evaluate (in-place bottom half, aggregate-first last
    layer over the evaluated rows in chunks) used when full_forward's
    workspace does not fit"""
    monkeypatch.setattr(mnn, "_full_fits", lambda g, st: False)
    g = epoch_graph(G, str(G[f"eval/{tag}/graph"]))
    dg = mq.DeviceGraph.from_csr(g, device="cuda:0")
    for phase in (0, 1):
        p = f"eval/{tag}/p{phase}"
        ws = [G[f"{p}/w{l}"] for l in range(3) if f"{p}/w{l}" in G]
        state = mq.ModelState(ws, device="cuda:0")
        for mask, key in ((g.val_mask, "val_acc"), (g.test_mask, "test_acc")):
            acc = mnn.evaluate(dg, state, mask, chunk=97)  # several chunks
            assert abs(acc - float(G[f"{p}/{key}"][0])) <= 0.005 + 1e-12, (key, acc)


def test_full_forward_cfg1_shape():
    from conftest import make_cfg1
    g = make_cfg1()
    dg = mq.DeviceGraph.from_csr(g, device="cuda:0")
    state = mq.init_model(64, 64, 4, num_layers=2, seed=0, device="cuda:0")
    ws = [w.cpu().numpy() for w in state.weights]
    ref = onn.full_forward(g.row_offsets, g.col_indices, g.features, ws)
    close_normwise(mnn.full_forward(dg, state).cpu().numpy(), ref)


# ------------------------------------------------------------ cache refresh
REFRESH = sorted({k.split("/")[2] for k in G if k.startswith("refresh/case/")})


@pytest.fixture(scope="module")
def g2_dev():
    return mq.DeviceGraph.from_csr(epoch_graph(G, "g2"), device="cuda:0")


def test_cache_probs_bit_exact(g2_dev):
    assert g2_dev.self_loops > 0
    got = mq.cache_probs_degree(g2_dev).cpu().numpy()
    assert np.array_equal(got, G["refresh/g2/degree_probs"])
    for fo, steps in ((5, 2), (10, 3)):
        got = mq.cache_probs_walk(g2_dev, fo, steps).cpu().numpy()
        assert np.array_equal(got, G[f"refresh/g2/walk_probs_f{fo}_s{steps}"]), (fo, steps)
    g = epoch_graph(G, "g2")
    g.train_mask = G["refresh/g2small/train_mask"]
    small = mq.DeviceGraph.from_csr(g, device="cuda:0")
    got = mq.cache_probs_walk(small, 2, 1).cpu().numpy()
    assert np.array_equal(got, G["refresh/g2small/walk_probs_f2_s1"])


@pytest.mark.parametrize("name", REFRESH)
def test_refresh_matches_reference(g2_dev, name):
    p = f"refresh/case/{name}"
    probs = G[str(G[f"{p}/probs_key"])]
    frac, seed, epoch = G[f"{p}/params"]
    cache = mq.refresh_cache(g2_dev, torch.as_tensor(probs), float(frac),
                             mq.RefreshStream(int(seed), int(epoch)))
    got = cache.cached_ids.cpu().numpy()
    assert np.array_equal(got, G[f"{p}/cached_ids"])


@pytest.mark.parametrize("frac,seed", [(0.01, 0), (0.1, 5), (0.5, 2)])
def test_refresh_cfg1_matches_oracle(frac, seed):
    from conftest import make_cfg1
    from oracle import cache as ocache
    from oracle.philox import RefreshRng
    g = make_cfg1()
    dg = mq.DeviceGraph.from_csr(g, device="cuda:0")
    for probs in (mq.cache_probs_degree(dg), mq.cache_probs_walk(dg, 10, 2)):
        p = probs.cpu().numpy()
        ref = ocache.refresh_cache_ids(g.num_nodes, p, frac, RefreshRng(seed, 3))
        got = mq.refresh_mask(dg, probs, frac, mq.RefreshStream(seed, 3)).cpu().numpy()
        assert np.array_equal(np.flatnonzero(got), ref)
    assert np.array_equal(mq.cache_probs_degree(dg).cpu().numpy(),
                          ocache.degree_probs(g.col_indices, g.num_nodes))
    assert np.array_equal(mq.cache_probs_walk(dg, 10, 2).cpu().numpy(),
                          ocache.walk_probs(g.row_offsets, g.col_indices, g.train_mask, 10, 2))


def test_refresh_odd_node_count_matches_oracle():
    """odd n exercises the scratch alignment; hubs, isolated rows and loops."""
    from oracle import cache as ocache
    from oracle.philox import RefreshRng
    g = _hub_graph(n=6001)
    g.train_mask = np.zeros(g.num_nodes, bool)
    g.train_mask[::3] = True
    dg = mq.DeviceGraph.from_csr(g, device="cuda:0")
    for probs in (mq.cache_probs_degree(dg), mq.cache_probs_walk(dg, 5, 2)):
        p = probs.cpu().numpy()
        for frac in (0.013, 0.2):
            ref = ocache.refresh_cache_ids(g.num_nodes, p, frac, RefreshRng(11, 2))
            got = mq.refresh_mask(dg, probs, frac, mq.RefreshStream(11, 2)).cpu().numpy()
            assert np.array_equal(np.flatnonzero(got), ref)
    assert np.array_equal(mq.cache_probs_walk(dg, 5, 2).cpu().numpy(),
                          ocache.walk_probs(g.row_offsets, g.col_indices, g.train_mask, 5, 2))


# ------------------------------------------------------------ graph ingest
@pytest.mark.parametrize("name", ["g8", "rand", "hub"])
def test_build_csr_matches_reference(name):
    g = mq.build_csr(G[f"ingest/{name}/edges"], int(G[f"ingest/{name}/n"][0]), device="cuda:0")
    assert np.array_equal(g.row_offsets.cpu().numpy(), G[f"ingest/{name}/row_offsets"])
    assert np.array_equal(g.col_indices.cpu().numpy().astype(np.int64),
                          G[f"ingest/{name}/col_indices"])
    assert np.array_equal(g.features.cpu().numpy(), G[f"ingest/{name}/features"])
    mq.DeviceGraph.from_csr(g, device="cuda:0")  # usable as is


def test_build_csr_large_and_errors():
    """several radix passes and many tiles against np.unique; range errors"""
    from oracle.sampler import build_csr as obuild
    rng = np.random.default_rng(5)
    n = 3_000_017
    e = rng.integers(0, n, size=(5_000_000, 2))
    e[::7] = e[::7][:, ::-1]
    e = np.concatenate([e, e[:100_000]])
    g = mq.build_csr(e, n, features=np.zeros((n, 4), np.float32), device="cuda:0")
    ro, col = obuild(e, n)
    assert np.array_equal(g.row_offsets.cpu().numpy(), ro)
    assert np.array_equal(g.col_indices.cpu().numpy().astype(np.int64), col)
    with pytest.raises(ValueError):
        mq.build_csr(np.array([[0, 5]]), 5, device="cuda:0")


def test_load_reference_container(tmp_path):
    p = tmp_path / "g2.mqg1"
    p.write_bytes(G["ingest/mqg1"].tobytes())
    g = mq.load(str(p), device="cuda:0")
    assert np.array_equal(g.row_offsets.cpu().numpy(), G["g2/row_offsets"])
    assert np.array_equal(g.col_indices.cpu().numpy().astype(np.int64), G["g2/col_indices"])
    assert np.array_equal(g.features.cpu().numpy(), G["g2/features"])
    assert np.array_equal(g.labels.cpu().numpy(), G["g2/labels"])
    for k in ("train_mask", "val_mask", "test_mask"):
        assert np.array_equal(getattr(g, k), G[f"g2/{k}"])
    bad = bytearray(G["ingest/mqg1"].tobytes())
    bad[:4] = b"XXXX"
    (tmp_path / "bad.mqg1").write_bytes(bytes(bad))
    with pytest.raises(ValueError):
        mq.load(str(tmp_path / "bad.mqg1"), device="cuda:0")
