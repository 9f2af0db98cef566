"""GPU parity of the PRODUCTION prep pass (mq_prep_batches: setup_q, sample_q,
the relabel chain, gather_q, labels_q) — the kernels StepRunner, run_epoch
and bench.py actually time — against the reference's own digests and the
oracle, slot by slot.

* every golden batch (tests/golden/sampling.npz: the g8 edge cases, g2 x
  {no cache, 1 %, 10 %} x {(10,5), (3,3,2), (1,)}, cfg1) is staged into a
  slot of a Q = 8 group next to other batches, the group is prepared in ONE
  pass and each slot's MiniBatch digest (targets, per-layer rows / cols /
  f64 values / src_ids / dst_ids, gathered f32 features) must equal the
  reference SHA-256 (samplers.py:63-72); labels and the hit/miss counters
  must equal the reference's too;
* the device batch plan (perm + cursor, runtime.py:95-117 round-robin deal)
  must cut the same batches as the host plan;
* at full size (Reddit-shaped configs[1] and products-shaped configs[2],
  test_gpu_prep_fullsize) every slot of a device-planned group is compared
  array-equal with oracle.sampler.build_minibatch.
"""

import numpy as np
import pytest

from conftest import batch_prefixes, golden_batch, make_cfg1, make_g2, make_g8

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2601_04707_b200 as mq  # noqa: E402
from oracle import sampler as osamp  # noqa: E402
from paper_2601_04707_b200.prep import PrepGroup, PrepShared  # noqa: E402

Q = 8


@pytest.fixture(scope="module")
def hosts(golden_sampling):
    return {"g8": make_g8(), "g2": make_g2(golden_sampling), "cfg1": make_cfg1()}


def _gname(prefix):
    return "g8" if prefix.startswith("g8") else "g2" if prefix.startswith("g2") else "cfg1"


def _groups(golden):
    """golden batches grouped by (graph, fanouts, cache mask)."""
    out = {}
    for p in batch_prefixes(golden):
        fo = tuple(int(x) for x in golden[f"{p}/fanouts"])
        key = (_gname(p), fo, str(golden[f"{p}/mask_name"]))
        out.setdefault(key, []).append(p)
    return out


def _run_group(g, cache, fanouts, batches, seed, epoch, placement_cache=None):
    """Stage [(bid, targets)] into one Q-slot group, prepare it in one pass."""
    bs = max(int(np.asarray(t).size) for _, t in batches)
    shared = PrepShared(g, fanouts, bs, Q)
    grp = PrepGroup(g, fanouts, bs, Q, shared)
    grp.stage(batches, seed, epoch)
    if cache is not None:
        cache.hit_miss.zero_()
    desc = grp.desc(cache, None, None, 1, 0)
    grp.launch(desc, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    return grp


@pytest.fixture(params=["direct", "hash"])
def rank_table(request, monkeypatch):
    """The relabel's rank words node-indexed, or hashed (the papers-scale
    layout, forced here on the small golden graphs)."""
    monkeypatch.setenv("MQ_PREP_HASH", "1" if request.param == "hash" else "0")
    return request.param


def _table_at_rest(grp):
    t = grp.shared.tbl
    if grp.shared.hash_lg:
        cap = 1 << grp.shared.hash_lg
        assert int(t[:, 0:2 * cap:2].abs().sum()) == 0  # every key empty again
        assert bool((t[:, 1:2 * cap:2] == 2 ** 31 - 1).all())
    else:
        assert bool((t == 2 ** 31 - 1).all())


def test_prep_pass_matches_reference_digests(golden_sampling, hosts, rank_table):
    """Every golden batch, prepared by the batched production pass in a full
    group of 8 slots (the group's other slots hold other batches of the same
    graph, or the same batches under other slots), reproduces the reference's
    digest, labels and hit/miss counts; the rank words are back at rest."""
    gs = golden_sampling
    devs = {k: mq.DeviceGraph.from_csr(h) for k, h in hosts.items()}
    checked = 0
    for (gname, fo, mask_name), prefixes in _groups(gs).items():
        g = devs[gname]
        cache = mq.DeviceCache(g, gs[mask_name]) if mask_name else None
        # one key per group (the prep pass keys slots by (seed, epoch, batch)):
        # split the prefixes by their (seed, epoch)
        by_key = {}
        for p in prefixes:
            seed, epoch, bid = (int(x) for x in gs[f"{p}/key"])
            by_key.setdefault((seed, epoch), []).append((bid, p))
        for (seed, epoch), items in by_key.items():
            # fill all Q slots: the batches, then the same batches again in
            # other slot positions (slots must not interfere)
            order = [items[i % len(items)] for i in range(Q)]
            batches = [(bid, gs[f"{p}/targets"]) for bid, p in order]
            grp = _run_group(g, cache, fo, batches, seed, epoch)
            assert (grp.shared.hash_lg > 0) == (rank_table == "hash")
            _table_at_rest(grp)
            tot_hits = tot_miss = 0
            for q, (bid, p) in enumerate(order):
                targets, layers, digest, hits = golden_batch(gs, p)
                mb = grp.minibatch(q, epoch)
                for l, ref in enumerate(layers):
                    r = mb.layers[l].to_reference()
                    for k in ("rows", "cols", "values", "src_ids", "dst_ids"):
                        assert np.array_equal(r[k], ref[k]), (p, q, l, k)
                assert np.array_equal(mb.target_labels.cpu().numpy(), gs[f"{p}/labels"]), (p, q)
                assert mb.digest() == digest, (p, q)
                tot_hits += int(hits[0])
                tot_miss += int(hits[1])
                checked += 1
            if cache is not None:
                assert [int(cache.hit_miss[0]), int(cache.hit_miss[1])] == [tot_hits, tot_miss]
    assert checked >= 8 * 10


def test_prep_pass_host_feature_store(golden_sampling, hosts):
    """Misses served from the pinned-host feature store (configs[3]'s
    host-miss path), hits from the HBM cache table: same digests."""
    gs = golden_sampling
    g = mq.DeviceGraph.from_csr(hosts["g2"], feature_placement="host")
    assert g.features.is_pinned()
    cache = mq.DeviceCache(g, gs["g2/mask10"])
    items = [p for p in batch_prefixes(gs) if p.startswith("g2_c10_10x5")]
    order = [items[i % len(items)] for i in range(Q)]
    seed, epoch, _ = (int(x) for x in gs[f"{order[0]}/key"])
    batches = [(int(gs[f"{p}/key"][2]), gs[f"{p}/targets"]) for p in order]
    grp = _run_group(g, cache, (10, 5), batches, seed, epoch)
    for q, p in enumerate(order):
        assert grp.minibatch(q, epoch).digest() == bytes(gs[f"{p}/digest"]).hex(), (p, q)


def test_prep_partial_group_and_empty_slots(golden_sampling, hosts):
    """A group with fewer batches than slots (the epoch's ragged tail): the
    staged slots still match, the empty ones produce empty blocks."""
    gs = golden_sampling
    g = mq.DeviceGraph.from_csr(hosts["g2"])
    cache = mq.DeviceCache(g, gs["g2/mask1"])
    p = "g2_c1_3x3x2_b1"
    seed, epoch, bid = (int(x) for x in gs[f"{p}/key"])
    grp = _run_group(g, cache, (3, 3, 2), [(bid, gs[f"{p}/targets"])], seed, epoch)
    assert grp.minibatch(0, epoch).digest() == bytes(gs[f"{p}/digest"]).hex()
    for q in range(1, Q):
        assert int(grp.hops[-1].counts[q, 0]) == 0 and int(grp.hops[-1].counts[q, 1]) == 0


def _device_plan_vs_oracle(hg, g, cache, mask, fanouts, batch_size, seed, epoch, world=1, rank=0,
                           check_slots=Q, group=None):
    """Production device plan (setup_q: perm + cursor) for one group; every
    slot compared array-equal with oracle.build_minibatch."""
    perm = mq.runtime.epoch_permutation(hg.train_mask, seed, epoch)
    shared = PrepShared(g, fanouts, batch_size, Q)
    grp = group or PrepGroup(g, fanouts, batch_size, Q, shared)
    grp.set_key(seed, epoch)
    dperm = torch.as_tensor(perm.astype(np.int32), device=g.device)
    cursor = torch.zeros(2, dtype=torch.int32, device=g.device)
    grp.launch(grp.desc(cache, dperm, cursor, world, rank), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert int(cursor[0]) == Q and int(cursor[1]) == 0
    ro = hg.row_offsets
    col = hg.col_indices
    feats = hg.features
    for q in range(check_slots):
        j = q * world + rank
        tg = perm[j * batch_size:(j + 1) * batch_size]
        if tg.size == 0:
            assert int(grp.n_targets[q, 0]) == 0
            continue
        ref = osamp.build_minibatch(ro, col, feats, hg.labels, tg, fanouts, seed=seed,
                                    epoch=epoch, batch_id=j, cached_mask=mask)
        mb = grp.minibatch(q, epoch)
        assert mb.batch_id == j
        assert np.array_equal(mb.target_ids.cpu().numpy(), tg)
        assert np.array_equal(mb.target_labels.cpu().numpy(), ref.target_labels)
        for l, rb in enumerate(ref.layers):
            r = mb.layers[l].to_reference()
            for k in ("rows", "cols", "values", "src_ids", "dst_ids"):
                assert np.array_equal(r[k], getattr(rb, k)), (q, l, k)
        assert np.array_equal(mb.features.cpu().numpy(), ref.features), q
        assert mb.digest() == ref.digest(), q
    return grp


@pytest.mark.parametrize("world,rank", [(1, 0), (3, 2)])
def test_device_plan_cfg1_vs_oracle(world, rank):
    """configs[0] (cfg1): the device-sliced round-robin deal of one epoch's
    permutation, 8 batches of 1024 prepared in one pass, vs the oracle."""
    hg = make_cfg1()
    g = mq.DeviceGraph.from_csr(hg)
    from paper_2601_04707_b200 import synth
    mask = synth.degree_cache_mask(torch.as_tensor(hg.col_indices), hg.num_nodes,
                                   0.01).cpu().numpy()
    cache = mq.DeviceCache(g, mask)
    _device_plan_vs_oracle(hg, g, cache, mask, (10, 5), 1024, seed=3, epoch=1, world=world,
                           rank=rank)
