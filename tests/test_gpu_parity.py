"""GPU parity: the CUDA path (through the C-ABI) against the reference-made
golden vectors and the CPU oracle.

Bars: sampling, relabel, gather, SpMM-forward and the
optimizer update are bit-exact; GEMM-based outputs and gradients are
tolerance-matched normwise: max|a-b| <= 1e-5 * max|b| (+ tiny absolute).
"""

import json

import numpy as np
import pytest

from conftest import (GOLDEN, batch_prefixes, golden_batch, make_cfg1, make_g2, make_g8)

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

from oracle import nn as onn  # noqa: E402
from oracle import sampler as osamp  # noqa: E402
from paper_2601_04707_b200 import nn as mnn  # noqa: E402
from paper_2601_04707_b200._lib import lib, ptr  # noqa: E402
from paper_2601_04707_b200.cache import DeviceCache, gather_features  # noqa: E402
from paper_2601_04707_b200.graph import DeviceGraph  # noqa: E402
from paper_2601_04707_b200.samplers import (PhiloxStream, SamplerParams,  # noqa: E402
                                            build_minibatch, node_wise_block)

RTOL = 1e-5


def assert_close_normwise(got, ref, rtol=RTOL, what=""):
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    assert got.shape == ref.shape, (what, got.shape, ref.shape)
    scale = max(np.abs(ref).max(initial=0.0), 1e-30)
    err = np.abs(got - ref).max(initial=0.0)
    assert err <= rtol * scale + 1e-30, f"{what}: max err {err:.3e} vs scale {scale:.3e}"


@pytest.fixture(scope="module")
def graphs(golden_sampling):
    return {"g8": DeviceGraph.from_csr(make_g8()),
            "g2": DeviceGraph.from_csr(make_g2(golden_sampling)),
            "cfg1": DeviceGraph.from_csr(make_cfg1())}


def _gname(prefix):
    return "g8" if prefix.startswith("g8") else "g2" if prefix.startswith("g2") else "cfg1"


def test_philox_device_matches_host_and_golden():
    kat = json.loads((GOLDEN / "philox_kat.json").read_text())
    for s in kat["streams"]:
        out = torch.zeros(s["k"], dtype=torch.int32, device="cuda")
        lib().mq_philox_fill(s["seed"], s["epoch"], s["batch"], s["hop"], s["row"], s["k"],
                             ptr(out), torch.cuda.current_stream().cuda_stream)
        got = (out.cpu().numpy().view(np.uint32)).tolist()
        assert got == s["draws"]
        pos = (np.zeros(s["k"], dtype=np.int64))
        lib().mq_fisher_yates_host(s["seed"], s["epoch"], s["batch"], s["hop"], s["row"], s["n"],
                                   s["k"], pos.ctypes.data)
        assert pos.tolist() == s["positions"]


def test_sampling_bit_exact_vs_reference_digests(golden_sampling, graphs):
    g = golden_sampling
    prefixes = batch_prefixes(g)
    caches = {}
    for p in prefixes:
        dg = graphs[_gname(p)]
        seed, epoch, bid = (int(x) for x in g[f"{p}/key"])
        mask_name = str(g[f"{p}/mask_name"])
        cache = None
        if mask_name:
            cache = caches.get(mask_name) or DeviceCache(dg, g[mask_name])
            caches[mask_name] = cache
        targets, layers, digest, hits = golden_batch(g, p)
        fo = tuple(int(x) for x in g[f"{p}/fanouts"])
        mb = build_minibatch(dg, targets, SamplerParams("sage", fo, num_layers=len(fo)),
                             PhiloxStream(seed, epoch, bid), batch_id=bid, epoch=epoch,
                             cached_mask=cache)
        for l, ref in enumerate(layers):
            r = mb.layers[l].to_reference()
            for k in ("rows", "cols", "values", "src_ids", "dst_ids"):
                assert np.array_equal(r[k], ref[k]), (p, l, k)
        assert mb.digest() == digest, p
        assert [mb.cache_hits, mb.cache_misses] == list(hits), p


@pytest.mark.parametrize("hop", [0, 1, 3])
def test_node_wise_block_any_hop_vs_oracle(golden_sampling, graphs, hop):
    g2 = make_g2(golden_sampling)
    dg = graphs["g2"]
    cache = DeviceCache(dg, golden_sampling["g2/mask10"])
    rng = np.random.default_rng(hop)
    for fanout in (1, 2, 7, 16, 25, 32):
        dst = rng.choice(2000, size=300, replace=False)
        for mask, c in ((None, None), (golden_sampling["g2/mask10"], cache)):
            blk = node_wise_block(dg, dst, fanout, PhiloxStream(5, 6, 7, hop), arch="sage", cached_mask=c)
            ref = osamp.node_wise_block(g2.row_offsets, g2.col_indices, dst, fanout, seed=5,
                                        epoch=6, batch_id=7, hop=hop, cached_mask=mask)
            r = blk.to_reference()
            for k in ("rows", "cols", "values", "src_ids"):
                assert np.array_equal(r[k], getattr(ref, k)), (fanout, k)


def test_duplicate_targets_and_empty_rows(graphs):
    """Duplicates keep their positions, the last occurrence owns the column
    (samplers.py:155-156); rows without neighbours emit nothing."""
    from conftest import HostGraph, csr_from_edges
    ro, col = csr_from_edges([(0, 1), (1, 0), (1, 2), (2, 1), (3, 3)], 5)  # 3: loop only, 4: none
    hg = HostGraph(ro, col, np.eye(5, 4, dtype=np.float32), np.zeros(5, np.int32), 2)
    dg = DeviceGraph.from_csr(hg)
    tg = np.array([1, 3, 4, 1, 0])
    blk = node_wise_block(dg, tg, 2, PhiloxStream(1, 2, 3), arch="sage")
    ref = osamp.node_wise_block(hg.row_offsets, hg.col_indices, tg, 2, seed=1, epoch=2,
                                batch_id=3, hop=0)
    r = blk.to_reference()
    for k in ("rows", "cols", "values", "src_ids"):
        assert np.array_equal(r[k], getattr(ref, k)), k


def test_gather_bit_exact_and_hit_routing(golden_cache, golden_sampling, graphs):
    gc = golden_cache
    dg = graphs["g2"]
    cache = DeviceCache(dg, gc["mask"])
    assert np.array_equal(cache.cached_ids.cpu().numpy(), gc["cached_ids"])
    out = gather_features(cache, dg, gc["ids"], count_hits=True)
    assert np.array_equal(out.cpu().numpy(), gc["gather"])
    assert int(cache.hit_miss[0]) == gc["hits"].size and int(cache.hit_miss[1]) == gc["misses"].size
    cache.table[:cache.size, :dg.feature_dim] += 100.0  # hits must come from the cache copy
    out = gather_features(cache, dg, gc["ids"])
    assert np.array_equal(out.cpu().numpy(), gc["gather_marked"])


def test_gather_host_miss_path(golden_cache, golden_sampling):
    gc = golden_cache
    dg = DeviceGraph.from_csr(make_g2(golden_sampling), feature_placement="host")
    assert dg.features.is_pinned()
    cache = DeviceCache(dg, gc["mask"])
    out = gather_features(cache, dg, gc["ids"])
    assert np.array_equal(out.cpu().numpy(), gc["gather"])


@pytest.mark.parametrize("tag", ["2l", "3l"])
def test_numerics_vs_reference(golden_nn, golden_sampling, graphs, tag):
    gn, gs = golden_nn, golden_sampling
    dg = graphs["g2"]
    cache = DeviceCache(dg, gs["g2/mask10"])
    fo = tuple(int(x) for x in gn[f"{tag}/fanouts"])
    hidden = int(gn[f"{tag}/hidden"][0])
    state = mnn.init_model(16, hidden, 5, num_layers=len(fo), seed=7, learning_rate=0.01)
    params = SamplerParams("sage", fo, num_layers=len(fo))
    for step in range(3):
        p = f"{tag}/s{step}"
        # start every step from the reference's weights so tolerances do not compound
        ref_state = [gn[f"{p}/w_before{l}"] for l in range(len(fo))]
        for l, w in enumerate(ref_state):
            state.weights[l].copy_(torch.as_tensor(w))
        mb = build_minibatch(dg, gn[f"{p}/targets"], params, PhiloxStream(4, 0, step),
                             batch_id=step, cached_mask=cache)
        logits, fc = mnn.forward(mb, state, return_cache=True)
        # layer-0 aggregation is bit-exact (np.add.at order)
        agg0 = fc["inputs"][0][1][:mb.layers[0].num_dst, :16].cpu().numpy()
        assert np.array_equal(agg0, gn[f"{p}/agg0"])
        assert_close_normwise(logits.cpu().numpy(), gn[f"{p}/logits"], what="logits")
        loss, dl = mnn.batch_loss(logits, mb.target_labels)
        assert loss == pytest.approx(float(gn[f"{p}/loss"][0]), rel=1e-5)
        assert_close_normwise(dl.cpu().numpy(), gn[f"{p}/dlogits"], what="dlogits")
        grads = mnn.backward(mb, state, fc, dl)
        for l, gr in enumerate(grads):
            assert_close_normwise(gr.cpu().numpy(), gn[f"{p}/grad{l}"], rtol=2e-5, what=f"grad{l}")


def test_adam_bit_exact_given_reference_grads(golden_nn):
    gn = golden_nn
    state = mnn.init_model(16, 32, 5, num_layers=2, seed=7, learning_rate=0.01)
    for step in range(3):
        p = f"2l/s{step}"
        mnn.adam_step(state, [torch.as_tensor(gn[f"{p}/grad{l}"]).cuda() for l in range(2)])
        for l in range(2):
            assert np.array_equal(state.weights[l].cpu().numpy(), gn[f"{p}/w_after{l}"]), (step, l)
            assert np.array_equal(state.m[l].cpu().numpy(), gn[f"{p}/m_after{l}"])
            assert np.array_equal(state.v[l].cpu().numpy(), gn[f"{p}/v_after{l}"])
    assert state.step_count == 3


def test_sgd_bit_exact(golden_nn):
    state = mnn.init_model(16, 32, 5, num_layers=2, seed=7, learning_rate=0.05)
    mnn.sgd_step(state, [torch.as_tensor(golden_nn[f"2l/s0/grad{l}"]).cuda() for l in range(2)])
    for l in range(2):
        assert np.array_equal(state.weights[l].cpu().numpy(), golden_nn[f"sgd/w_after{l}"])


def test_spmm_backward_vs_oracle(golden_sampling, graphs):
    """block_apply_t + self add on a real block (fp32 atomics: normwise 1e-6)."""
    gs = golden_sampling
    dg = graphs["g2"]
    _, layers, _, _ = golden_batch(gs, "g2_c10_10x5_b0")
    ref_blk = layers[1]  # hop-0 block (dst = targets)

    class B:
        pass
    b = B()
    b.rows, b.cols, b.values = ref_blk["rows"], ref_blk["cols"], ref_blk["values"]
    b.num_dst, b.num_src = ref_blk["dst_ids"].size, ref_blk["src_ids"].size
    b.dst_in_src = np.arange(b.num_dst)
    d = 24
    rng = np.random.default_rng(3)
    dt = rng.standard_normal((b.num_dst, 2 * d)).astype(np.float32)
    ref = onn.block_apply_t(b, dt[:, :d], b.num_src)
    np.add.at(ref, b.dst_in_src, dt[:, d:])
    dev = dg.device
    rows = torch.as_tensor(b.rows, dtype=torch.int32, device=dev)
    cols = torch.as_tensor(b.cols, dtype=torch.int32, device=dev)
    vals = torch.as_tensor(b.values.astype(np.float32), device=dev)
    counts = torch.tensor([b.num_src, b.rows.size], dtype=torch.int32, device=dev)
    nd = torch.tensor([b.num_dst], dtype=torch.int32, device=dev)
    dtt = torch.as_tensor(dt, device=dev)
    dh = torch.empty((b.num_src, d), dtype=torch.float32, device=dev)
    lib().mq_spmm_bwd(ptr(rows), ptr(cols), ptr(vals), ptr(counts), b.rows.size, ptr(nd),
                      b.num_src, ptr(dtt), 2 * d, d, None, 0, ptr(dh), d,
                      torch.cuda.current_stream().cuda_stream)
    assert_close_normwise(dh.cpu().numpy(), ref, rtol=1e-6, what="spmm_bwd")


def test_per_op_tcgen05_matches_ffma(golden_sampling, graphs):
    """The per-op SAGE transform / weight gradient on tcgen05 (3xTF32, split-K
    partials summed by mq_grad_reduce) against the FFMA split-K path at a
    wider hidden size, with a class count whose dlogits pitch (5) needs the
    16-byte-aligned copy."""
    dg = graphs["g2"]
    params = SamplerParams("sage", (10, 5, 3), num_layers=3)
    tg = np.random.default_rng(11).choice(2000, 512, replace=False)
    mb = build_minibatch(dg, tg, params, PhiloxStream(9, 0, 1), batch_id=1)
    state = mnn.init_model(16, 64, 5, num_layers=3, seed=3, learning_rate=0.01)
    out = {}
    old = lib().mq_get_gemm_backend()
    try:
        for be in (1, 0):
            lib().mq_set_gemm_backend(be)
            logits, fc = mnn.forward(mb, state, return_cache=True)
            loss, dl = mnn.batch_loss(logits, mb.target_labels)
            grads = mnn.backward(mb, state, fc, dl)
            out[be] = (logits.cpu().numpy(), loss, [g.cpu().numpy() for g in grads])
    finally:
        lib().mq_set_gemm_backend(old)
    assert_close_normwise(out[1][0], out[0][0], rtol=2e-5, what="logits")
    assert out[1][1] == pytest.approx(out[0][1], rel=1e-5)
    for l, (a, b) in enumerate(zip(out[1][2], out[0][2])):
        assert_close_normwise(a, b, rtol=2e-5, what=f"grad{l}")
