"""GPU: the seed-partitioned feature store (BASELINE configs[4]).

Node v's feature row lives on rank v % G at row v // G; the other ranks'
shards are mapped over NVLink (CUDA IPC).  Gathering through the shards must
be bit-identical to gathering from one replicated table:

* one process standing in for G = 1, 2, 3, 8 shards (use_local_shards): the
  production prep pass reproduces the reference's batch digests (gathered f32
  features included), the per-op gather_features and the GNS cache table
  match the replicated store;
* two processes on one GPU, each holding only its shard and mapping the
  other's through CUDA IPC (feature_placement="sharded", the generator
  producing only the rank's rows): whole epochs over the peer exchange equal
  the reference's run_epoch fixtures like the replicated runs do;
* full-graph evaluation refuses a sharded table (it reads every row).
"""

import contextlib
import os
import socket

import numpy as np
import pytest

from conftest import batch_prefixes, load_golden, make_g2

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import torch.multiprocessing as mp  # noqa: E402

import paper_2601_04707_b200 as mq  # noqa: E402
from paper_2601_04707_b200.prep import PrepGroup, PrepShared  # noqa: E402

Q = 8


@pytest.mark.parametrize("G", [1, 2, 3, 8])
def test_local_shards_reproduce_reference_digests(golden_sampling, G):
    gs = golden_sampling
    g = mq.DeviceGraph.from_csr(make_g2(gs))
    ref_feats = g.features.clone()
    g.use_local_shards(G)
    g.features = None  # every read must go through the shards
    cache = mq.DeviceCache(g, gs["g2/mask10"])
    ids = cache.cached_ids
    np.testing.assert_array_equal(cache.table[:cache.size].cpu().numpy(),
                                  ref_feats[ids].cpu().numpy())
    items = [p for p in batch_prefixes(gs) if p.startswith("g2_c10_10x5")]
    order = [items[i % len(items)] for i in range(Q)]
    seed, epoch, _ = (int(x) for x in gs[f"{order[0]}/key"])
    batches = [(int(gs[f"{p}/key"][2]), gs[f"{p}/targets"]) for p in order]
    bs = max(np.asarray(t).size for _, t in batches)
    grp = PrepGroup(g, (10, 5), bs, Q, PrepShared(g, (10, 5), bs, Q))
    grp.stage(batches, seed, epoch)
    grp.launch(grp.desc(cache, None, None, 1, 0), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    for q, p in enumerate(order):
        assert grp.minibatch(q, epoch).digest() == bytes(gs[f"{p}/digest"]).hex(), (G, p, q)
    # per-op gather_features (misses from the shards, hits from the cache)
    rng = np.random.default_rng(G)
    some = rng.integers(0, g.num_nodes, 777)
    for c in (None, cache):
        out = mq.gather_features(c, g, some)
        np.testing.assert_array_equal(out.cpu().numpy(),
                                      ref_feats[torch.as_tensor(some)][:, :g.feature_dim]
                                      .cpu().numpy())
    with pytest.raises(NotImplementedError):
        mq.full_forward(g, mq.init_model(16, 16, 5, num_layers=2, seed=5))


def _free_port():
    with contextlib.closing(socket.socket(socket.AF_INET, socket.SOCK_STREAM)) as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        gs, rt = load_golden("sampling.npz"), load_golden("runtime.npz")
        hg = make_g2(gs)
        hg.train_mask = rt["epoch/train_mask"]
        hg.features = hg.features[rank::world].copy()  # this rank's rows only
        g = mq.DeviceGraph.from_csr(hg, feature_placement="sharded")
        assert g.features is None and len(g.shards) == world
        cache = mq.DeviceCache(g, gs["g2/mask10"])
        rep = mq.init_model(16, 16, 5, num_layers=2, seed=5, learning_rate=0.01)
        cfg = mq.PipelineConfig(num_devices=world, batch_size=64,
                                sampler=mq.SamplerParams("sage", (4, 3), num_layers=2),
                                optimizer="adam", sync_period=1, seed=5, exchange="peer")
        st, _ = mq.run_epoch(g, cache, [rep], cfg, epoch=1)
        bids = sorted(st.losses)
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), bids=np.array(bids),
                 losses=np.array([st.losses[b] for b in bids]),
                 hits=np.array([st.cache_hits, st.cache_misses]),
                 w0=rep.weights[0].cpu().numpy(), w1=rep.weights[1].cpu().numpy())
    finally:
        dist.destroy_process_group()


def test_two_ranks_sharded_store_match_reference_epoch(tmp_path):
    rt = load_golden("runtime.npz")
    mp.start_processes(_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True,
                       start_method="spawn")
    res = [np.load(tmp_path / f"rank{r}.npz") for r in range(2)]
    name = "2dev_adam"
    assert res[0]["bids"].tolist() == rt[f"epoch/{name}/loss_bids"].tolist()
    np.testing.assert_allclose(res[0]["losses"], rt[f"epoch/{name}/losses"], rtol=1e-4)
    assert res[0]["hits"].tolist() == rt[f"epoch/{name}/hits"].tolist()
    for l in range(2):
        w = rt[f"epoch/{name}/w{l}"]
        assert np.abs(res[0][f"w{l}"] - w).max() <= 1e-4 * np.abs(w).max()
        np.testing.assert_array_equal(res[1][f"w{l}"], res[0][f"w{l}"])
