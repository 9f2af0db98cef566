"""GPU: the multi-process RaCoM path (one process per "device", DistExchange
over torch.distributed) on real device kernels.  Only one GPU is available to
this build, so both ranks share cuda:0 and talk over gloo (the production
launcher uses NCCL, one GPU per rank; the exchange code is the same).

The 2-rank run must reproduce the single-process 2-replica run (LocalExchange,
the reference's in-process device threads) to the bar of the reference's
acceptance criterion 03 (1e-6): the f64 window all-reduce of two
contributions is order-free, and what remains is the fp32 atomic scatter
order of the backward (run-to-run noise).  The two ranks end the epoch with
bit-identical replicas (the epoch-barrier model average)."""

import contextlib
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import torch.multiprocessing as mp  # noqa: E402

from conftest import load_golden, make_g2  # noqa: E402


def _free_port():
    with contextlib.closing(socket.socket(socket.AF_INET, socket.SOCK_STREAM)) as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _config(mq, sync_period, optimizer):
    return mq.PipelineConfig(num_devices=2, batch_size=100,
                             sampler=mq.SamplerParams("sage", (5, 3), num_layers=2),
                             optimizer=optimizer, seed=4, sync_period=sync_period)


def _worker(rank, port, sync_period, optimizer, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE="2")
    import torch.distributed as dist
    import paper_2601_04707_b200 as mq
    dist.init_process_group("gloo", rank=rank, world_size=2)
    try:
        gs = load_golden("sampling.npz")
        g = mq.DeviceGraph.from_csr(make_g2(gs), device="cuda:0")
        cache = mq.DeviceCache(g, gs["g2/mask10"])
        st = mq.init_model(16, 24, 5, num_layers=2, seed=9, learning_rate=0.01)
        stats = []
        for epoch in range(2):
            s, _ = mq.run_epoch(g, cache, [st], _config(mq, sync_period, optimizer), epoch=epoch)
            stats.append(s)
        w = [x.cpu().numpy() for x in st.weights]
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"),
                 losses=np.array([stats[e].losses[b] for e in range(2)
                                  for b in sorted(stats[e].losses)]),
                 syncs=np.array([s.sync_count for s in stats]), *w)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("sync_period,optimizer", [(1, "adam"), (3, "sgd")])
def test_two_ranks_match_two_replicas(tmp_path, sync_period, optimizer):
    import paper_2601_04707_b200 as mq
    gs = load_golden("sampling.npz")
    g = mq.DeviceGraph.from_csr(make_g2(gs), device="cuda:0")
    cache = mq.DeviceCache(g, gs["g2/mask10"])
    reps = [mq.init_model(16, 24, 5, num_layers=2, seed=9, learning_rate=0.01) for _ in range(2)]
    local = []
    for epoch in range(2):
        s, _ = mq.run_epoch(g, cache, reps, _config(mq, sync_period, optimizer), epoch=epoch)
        local.append(s)
    ref_losses = np.array([local[e].losses[b] for e in range(2) for b in sorted(local[e].losses)])
    ref_w = [x.cpu().numpy() for x in reps[0].weights]
    for a, b in zip(reps[0].weights, reps[1].weights):
        assert torch.equal(a, b)  # replicas identical after the epoch barrier

    mp.start_processes(_worker, args=(_free_port(), sync_period, optimizer, str(tmp_path)),
                       nprocs=2, join=True, start_method="spawn")
    out = [np.load(tmp_path / f"rank{rank}.npz") for rank in range(2)]
    for r in out:
        np.testing.assert_allclose(r["losses"], ref_losses, rtol=1e-6)
        assert list(r["syncs"]) == [s.sync_count for s in local]
        for l, w in enumerate(ref_w):
            assert np.abs(r[f"arr_{l}"] - w).max() <= 1e-6 * np.abs(w).max()
    for l in range(len(ref_w)):
        np.testing.assert_array_equal(out[0][f"arr_{l}"], out[1][f"arr_{l}"])
