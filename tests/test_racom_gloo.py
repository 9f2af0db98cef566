"""RaCoM over torch.distributed (gloo, world size 2, CPU) — no GPU needed.

The multi-GPU path shares its host logic (racom.WindowDriver, DistExchange,
the f64 [grads | contributor count] packing, milestone/epoch syncs) with
these tests; only the per-replica numerics differ.  Here every replica is an
oracle-backed runner, so the distributed schedule can be checked against the
single-process zero-delay reference schedule (acceptance criterion 03,
test_acceptance.py:119-167: async RaCoM with P=1, zero delay == synchronous
DP within 1e-6) and against the reference's own run_epoch golden vectors.
"""

import contextlib
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import load_golden, make_g2
from oracle import nn as onn
from oracle import racom as oracom
from oracle import sampler as osamp
from paper_2601_04707_b200.racom import DistExchange, LocalExchange, WindowDriver


class OracleRunner:
    """The runner protocol of racom.WindowDriver with oracle numerics."""

    def __init__(self, graph, model, *, fanouts, batch_size, seed, world, rank, optimizer,
                 cached_mask=None):
        self.g, self.model = graph, model
        self.fanouts, self.B, self.seed = fanouts, batch_size, seed
        self.world, self.rank, self.optimizer = world, rank, optimizer
        self.mask = cached_mask
        self.P = sum(w.size for w in model.weights)
        self.grad64 = torch.zeros(self.P + 1, dtype=torch.float64)
        self.windows_done = 0
        self.losses = {}

    def begin_epoch(self, epoch, perm):
        self.epoch, self.perm, self.windows_done = epoch, perm, 0

    def compute_window(self):
        j = self.windows_done * self.world + self.rank
        tg = self.perm[j * self.B:(j + 1) * self.B]
        if tg.size == 0:
            self.grad64.zero_()
            return
        g = self.g
        mb = osamp.build_minibatch(g["row_offsets"], g["col_indices"], g["features"], g["labels"],
                                   tg, self.fanouts, seed=self.seed, epoch=self.epoch, batch_id=j,
                                   cached_mask=self.mask)
        loss, grads, _ = onn.loss_and_grads(mb.layers, mb.features, mb.target_labels,
                                            self.model.weights)
        self.losses[j] = loss
        flat = np.concatenate([gr.astype(np.float64).ravel() for gr in grads] + [[1.0]])
        self.grad64.copy_(torch.from_numpy(flat))

    def apply_window(self):
        g = self.grad64.numpy()
        mean, off = [], 0
        for w in self.model.weights:
            mean.append((g[off:off + w.size] / g[self.P]).reshape(w.shape))
            off += w.size
        (onn.adam_step if self.optimizer == "adam" else onn.sgd_step)(self.model, mean)
        self.windows_done += 1

    def state64(self):
        parts = [np.concatenate([a.astype(np.float64).ravel() for a in getattr(self.model, k)])
                 for k in ("weights", "m", "v")]
        return torch.from_numpy(np.concatenate(parts))

    def load_state64(self, t, n):
        x = (t.numpy() / n)
        off = 0
        for k in ("weights", "m", "v"):
            for a in getattr(self.model, k):
                a[...] = x[off:off + a.size].reshape(a.shape).astype(a.dtype)
                off += a.size

    @property
    def step_count(self):
        return self.model.step_count

    def sync_point(self):
        pass

    def stream_ctx(self):
        return contextlib.nullcontext()

    def wait_current(self):
        pass


def _graph_dict(gs, train_mask):
    g = make_g2(gs)
    return dict(row_offsets=g.row_offsets, col_indices=g.col_indices, features=g.features,
                labels=g.labels, train_mask=train_mask)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, case, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        gs = load_golden("sampling.npz")
        rt = load_golden("runtime.npz")
        graph = _graph_dict(gs, rt["epoch/train_mask"])
        opt, P, B, mask_name = case
        model = onn.init_model(16, 16, 5, num_layers=2, seed=5, learning_rate=0.01)
        r = OracleRunner(graph, model, fanouts=(4, 3), batch_size=B, seed=5, world=world,
                         rank=rank, optimizer=opt, cached_mask=gs[mask_name] if mask_name else None)
        _, expected = oracom.plan_epoch(graph["train_mask"], world, B, 5, 1)
        perm = np.random.default_rng(np.random.SeedSequence([5, 1, 0])).permutation(
            np.flatnonzero(graph["train_mask"]))
        r.begin_epoch(1, perm)
        info = WindowDriver([r], DistExchange(), sync_period=P).run(len(expected))
        out_q.put((rank, [w.copy() for w in model.weights], r.losses, info))
    finally:
        dist.destroy_process_group()


def _run_dist(case, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return sorted(res, key=lambda x: x[0])


@pytest.mark.parametrize("case", [("sgd", 1, 64, None), ("adam", 1, 64, "g2/mask10"),
                                  ("sgd", 3, 64, None), ("adam", 2, 48, "g2/mask1")])
def test_gloo_racom_matches_serial_reference_schedule(case, golden_sampling, golden_runtime):
    opt, P, B, mask_name = case
    res = _run_dist(case)
    # replicas identical after the epoch barrier (test_runtime.py:174-186)
    for a, b in zip(res[0][1], res[1][1]):
        assert np.array_equal(a, b)
    # same numbers as the single-process serial schedule (crit. 03 bar: 1e-6)
    graph = _graph_dict(golden_sampling, golden_runtime["epoch/train_mask"])
    base = onn.init_model(16, 16, 5, num_layers=2, seed=5, learning_rate=0.01)
    models = [base.copy(), base.copy()]
    losses, _ = oracom.run_epoch_serial(graph, models, fanouts=(4, 3), batch_size=B, seed=5,
                                        epoch=1, optimizer=opt, sync_period=P,
                                        cached_mask=golden_sampling[mask_name] if mask_name else None)
    for a, b in zip(res[0][1], models[0].weights):
        assert np.abs(a - b).max() <= 1e-6
    got = {**res[0][2], **res[1][2]}
    assert sorted(got) == sorted(losses)
    for k in losses:
        assert got[k] == pytest.approx(losses[k], rel=1e-6)
    windows = res[0][3]["applied"]
    assert res[0][3]["sync_count"] == windows // P and res[0][3]["epoch_sync"] == 1


def test_gloo_matches_reference_run_epoch_golden(golden_sampling, golden_runtime):
    """2 ranks over gloo reproduce the reference's own 2-device run_epoch."""
    rt = golden_runtime
    res = _run_dist(("adam", 1, 64, "g2/mask10"))
    for l in range(2):
        w = rt[f"epoch/2dev_adam/w{l}"]
        assert np.abs(res[0][1][l] - w).max() <= 1e-6
    got = {**res[0][2], **res[1][2]}
    bids = rt["epoch/2dev_adam/loss_bids"].tolist()
    np.testing.assert_allclose([got[b] for b in bids], rt["epoch/2dev_adam/losses"], rtol=1e-6)


def test_local_exchange_equals_single_process_schedule(golden_sampling, golden_runtime):
    """Several replicas in one process (the reference's simulated devices)."""
    graph = _graph_dict(golden_sampling, golden_runtime["epoch/train_mask"])
    G, B = 3, 48
    base = onn.init_model(16, 16, 5, num_layers=2, seed=5, learning_rate=0.01)
    runners = [OracleRunner(graph, base.copy(), fanouts=(4, 3), batch_size=B, seed=5, world=G,
                            rank=r, optimizer="adam") for r in range(G)]
    perm = np.random.default_rng(np.random.SeedSequence([5, 1, 0])).permutation(
        np.flatnonzero(graph["train_mask"]))
    for r in runners:
        r.begin_epoch(1, perm)
    _, expected = oracom.plan_epoch(graph["train_mask"], G, B, 5, 1)
    assert expected[-1] < G  # ragged last window: fewer contributors
    info = WindowDriver(runners, None, sync_period=2).run(len(expected))
    models = [base.copy() for _ in range(G)]
    oracom.run_epoch_serial(graph, models, fanouts=(4, 3), batch_size=B, seed=5, epoch=1,
                            optimizer="adam", sync_period=2)
    for r in runners:
        for a, b in zip(r.model.weights, models[0].weights):
            assert np.abs(a - b).max() <= 1e-6
    assert info["epoch_sync"] == 1


def test_local_exchange_sums_in_replica_order():
    ts = [torch.tensor([1.0, 2.0], dtype=torch.float64), torch.tensor([3.0, 5.0], dtype=torch.float64)]
    LocalExchange(2).allreduce_sum_many(ts)
    assert ts[0].tolist() == [4.0, 7.0] == ts[1].tolist()


@pytest.mark.parametrize("P", [1, 2])
def test_sync_elision_is_exact(P, golden_sampling, golden_runtime):
    """Skipping the averages of provably identical replicas changes no bit:
    replicas seeded differently, first sync performed, later ones elided."""
    graph = _graph_dict(golden_sampling, golden_runtime["epoch/train_mask"])
    G, B = 3, 48
    perm = np.random.default_rng(np.random.SeedSequence([5, 1, 0])).permutation(
        np.flatnonzero(graph["train_mask"]))
    _, expected = oracom.plan_epoch(graph["train_mask"], G, B, 5, 1)
    out = {}
    for elide in (False, True):
        runners = [OracleRunner(graph, onn.init_model(16, 16, 5, num_layers=2, seed=5 + r,
                                                      learning_rate=0.01),
                                fanouts=(4, 3), batch_size=B, seed=5, world=G, rank=r,
                                optimizer="adam") for r in range(G)]
        for r in runners:
            r.begin_epoch(1, perm)
        info = WindowDriver(runners, None, sync_period=P, elide_identical=elide).run(len(expected))
        out[elide] = ([[w.copy() for w in r.model.weights] for r in runners], info)
    (w0, i0), (w1, i1) = out[False], out[True]
    assert i0["elided"] == 0 and i1["elided"] == i1["sync_count"] + i1["epoch_sync"] - 1 > 0
    assert i0["sync_count"] == i1["sync_count"]
    for ra, rb in zip(w0, w1):
        for a, b in zip(ra, rb):
            assert np.array_equal(a, b)
