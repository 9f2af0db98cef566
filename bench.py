#!/usr/bin/env python
"""Benchmark: seed nodes/s of MQ-GNN's per-iteration GraphSAGE training step.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--shape reddit|products|cfg1] [--no-cpu-baseline]

A step = one RaCoM window on every rank: device-side batch plan, 2 hops of
GNS-cache-biased sampling + relabel, feature gather, SAGE forward, summed
softmax-CE, backward, (f64 gradient all-reduce when N > 1) and Adam — the
per-batch body of the reference's run_epoch (mqpipe/runtime.py:294-323).

Workload (BASELINE.json configs[1]): Reddit-shaped synthetic power-law graph,
232,965 nodes, 114M arcs, 602-d features, 41 classes, fanouts [10, 5],
batch 1024, hidden 64, 1% degree-mode GNS cache, Adam lr 1e-3.  Graph,
features and cache are resident in HBM before timing (``value``); ``e2e``
is the same metric through the public host-buffer entry point
(StepRunner.step_from_host: pinned H2D of the batch's targets, one graph
launch, D2H of the loss, every step).  Inputs (1.1 GB of CSR + features)
exceed the 126 MB L2, so no explicit flush is done.

``--impl reference`` times the CPU oracle port of the reference path
(oracle/, restated from mqpipe and pinned to reference-generated golden
vectors) on this host's cores, on a bounded sample of the same workload.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "seed nodes/sec & epoch time at 1/2/4/8 B200; sample/gather/SpMM GB/s vs HBM"
UNIT = "seed nodes/s"
SHAPE_DESC = {
    "reddit": "reddit-shaped: 232,965 nodes / 114M arcs / 602-d / 41 classes, SAGE 2-layer "
              "fanout [10,5], batch 1024, hidden 64, 1% GNS degree cache (BASELINE configs[1])",
    "products": "ogbn-products-shaped: 2,449,029 nodes / 62M arcs / 100-d / 47 classes, SAGE "
                "3-layer fanout [15,10,5], batch 1024, hidden 64, 1% GNS walk-free degree cache",
    "cfg1": "cfg1: 10k nodes / 100k arcs / 64-d / 4 classes, SAGE 2-layer fanout [10,5], "
            "batch 1024, hidden 64, 1% GNS degree cache (BASELINE configs[0])",
    "papers": "ogbn-papers100M-shaped: 111M nodes / 1.6B arcs / 128-d / 172 classes, SAGE 3-layer "
              "fanout [15,10,5], batch 1024, hidden 64, 1% GNS walk cache, 1.1% train nodes "
              "(BASELINE configs[4], whole graph resident on each GPU)",
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1500)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--shape", default="reddit", choices=list(SHAPE_DESC))
    ap.add_argument("--batch", type=int, default=1024)
    ap.add_argument("--hidden", type=int, default=64)
    ap.add_argument("--cache-fraction", type=float, default=0.01)
    ap.add_argument("--feature-placement", default="hbm", choices=["hbm", "host", "sharded"],
                    help="feature table in HBM, pinned host memory, or node-partitioned "
                         "across the ranks (remote rows over NVLink P2P)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=20.0)
    ap.add_argument("--profile-steps", type=int, default=20,
                    help="launches per op in the per-kernel graph timing (0: skip)")
    ap.add_argument("--e2e-steps", type=int, default=600)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--queue-depth", default=None,
                    help="batches per batched prep pass (MQ-GNN queue depth Q), or 'auto'")
    ap.add_argument("--no-pdl", action="store_true", help="disable programmatic dependent launch")
    ap.add_argument("--layer0", default="auto", choices=["auto", "tf", "af"],
                    help="input layer transform-first / aggregate-first")
    ap.add_argument("--no-pipeline", action="store_true",
                    help="prep and train on one stream (no multi-queue overlap)")
    ap.add_argument("--exchange", default="peer", choices=["peer", "collective"],
                    help="N > 1: RaCoM over peer memory (in-graph) or a host-issued all-reduce")
    ap.add_argument("--staleness", type=int, default=0, choices=[0, 1],
                    help="N > 1 peer exchange: 0 parity schedule, 1 pipelined (one-window stale)")
    return ap.parse_args()


def env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


# --------------------------------------------------------------------- inputs
def build_inputs(args, device, feature_shard=None):
    """Synthetic graph (GPU generator when a GPU exists) + degree-mode cache mask;
    ``feature_shard=(G, r)`` generates only this rank's feature rows."""
    from paper_2601_04707_b200 import synth
    t0 = time.perf_counter()
    sg, fanouts = synth.generate_shape(args.shape, seed=args.seed, device=device,
                                       feature_shard=feature_shard)
    t_gen = time.perf_counter() - t0
    return sg, fanouts, t_gen


def oracle_cache_mask(ro, col, train_mask, fraction, seed, fanouts, epoch=0):
    """The reference's per-epoch residency on the CPU (oracle restatement of
    cache_probs_degree / cache_probs_walk / refresh_cache, cache.py:41-108, under
    the refresh injected-draw contract) — equal to the device refresh."""
    from oracle import cache as ocache
    from oracle.philox import RefreshRng
    n = ro.size - 1
    if float(np.mean(train_mask)) >= 0.5:
        probs = ocache.degree_probs(col, n)
    else:
        probs = ocache.walk_probs(ro, col, train_mask, fanouts[0], len(fanouts))
    ids = ocache.refresh_cache_ids(n, probs, fraction, RefreshRng(seed, epoch))
    mask = np.zeros(n, dtype=bool)
    mask[ids] = True
    return mask


def host_arrays(sg):
    import torch

    def h(a, dt):
        if isinstance(a, torch.Tensor):
            return a.detach().cpu().numpy().astype(dt, copy=False)
        return np.asarray(a).astype(dt, copy=False)
    return (h(sg.row_offsets, np.int64), h(sg.col_indices, np.int64),
            h(sg.features, np.float32), h(sg.labels, np.int32))


# ---------------------------------------------------------------- CPU oracle
_CPU = {}  # graph arrays shared with forked sampler workers (copy-on-write)


def _cpu_sample(j):
    """One batch's sample + relabel + gather (samplers.py:502-540) in a worker."""
    from oracle import sampler as osamp
    c = _CPU
    tg = c["perm"][j * c["B"]:(j + 1) * c["B"]]
    if tg.size == 0:
        return None
    return osamp.build_minibatch(c["ro"], c["col"], c["feats"], c["labels"], tg, c["fanouts"],
                                 seed=c["seed"], epoch=0, batch_id=c["bid0"] + j,
                                 cached_mask=c["mask"])


def cpu_oracle_run(ro, col, feats, labels, mask, perm, fanouts, args, budget_s, max_batches,
                   workers=None, bid0=0):
    """The reference's per-batch path on the host cores: like the reference's
    threaded runtime (runtime.py:413-577), sampler workers build batches in
    parallel (one process per spare core: the oracle is NumPy) while the main
    process runs forward/backward and Adam in batch order (oracle/ restatement
    of mqpipe, pinned to the reference's golden vectors).
    Returns (seeds, batches, seconds, cores used)."""
    import multiprocessing as mp
    from oracle import nn as onn
    model = onn.init_model(feats.shape[1], args.hidden, int(labels.max()) + 1,
                           num_layers=len(fanouts), seed=args.seed, learning_rate=1e-3)
    B = args.batch
    n_batches = min(max_batches, -(-len(perm) // B))
    if workers is None:
        workers = max(1, cores_used() - 1)
    _CPU.update(ro=ro, col=col, feats=feats, labels=labels, mask=mask, perm=perm, B=B,
                fanouts=fanouts, seed=args.seed, bid0=bid0)
    seeds = nb = 0
    t0 = time.perf_counter()
    t_fill = None  # steady state: the clock restarts once the first batch is applied
    pool = mp.get_context("fork").Pool(workers) if workers > 1 else None
    try:
        it = (pool.imap(_cpu_sample, range(n_batches), chunksize=1) if pool
              else map(_cpu_sample, range(n_batches)))
        for mb in it:
            if mb is None:
                break
            _, grads, _ = onn.loss_and_grads(mb.layers, mb.features, mb.target_labels,
                                             model.weights)
            onn.adam_step(model, grads)
            if t_fill is None and n_batches > 1:  # pool start-up + pipeline fill: not timed
                t_fill = time.perf_counter()
                continue
            seeds += mb.target_ids.size
            nb += 1
            if time.perf_counter() - t0 > budget_s:
                break
        dt = time.perf_counter() - (t_fill if t_fill is not None else t0)
    finally:
        if pool is not None:
            pool.terminate()
    return seeds, nb, dt, workers + 1 if pool else 1


def cores_used():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


# ------------------------------------------------------------------- clocks
class ClockSampler:
    """SM clock and throttle reasons sampled DURING the timed region: an NVML
    thread polls every ~2 ms (the Reddit timed region is ~70 ms, the driver's
    20-step run ~1 ms) and ``mark_start`` / ``mark_stop`` bracket the region
    on the host clock; nvidia-smi at 100 ms is the fallback."""
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.path = None
        self.thread = None
        self.samples = []  # (host time, sm MHz, reason bits)
        self.t0 = self.t1 = None

    def _handle(self, nv):
        try:  # the CUDA device's PCI address: NVML and CUDA indices may differ
            import torch
            pr = torch.cuda.get_device_properties(self.gpu)
            bus = f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
            return nv.nvmlDeviceGetHandleByPciBusId(bus)
        except Exception:
            return nv.nvmlDeviceGetHandleByIndex(self.gpu)

    def start(self):
        import threading
        try:
            import pynvml as nv
            nv.nvmlInit()
            h = self._handle(nv)
            self.max_mhz = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
            bits = {"hw_slowdown": nv.nvmlClocksThrottleReasonHwSlowdown,
                    "hw_thermal_slowdown": nv.nvmlClocksThrottleReasonHwThermalSlowdown,
                    "sw_thermal_slowdown": nv.nvmlClocksThrottleReasonSwThermalSlowdown,
                    "sw_power_cap": nv.nvmlClocksThrottleReasonSwPowerCap}
            self.bits = bits
            self.stop_flag = threading.Event()

            def loop():
                while not self.stop_flag.is_set():
                    try:
                        sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                        rs = nv.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                    except Exception:  # pragma: no cover
                        break
                    self.samples.append((time.perf_counter(), float(sm), int(rs)))
                    time.sleep(0.002)
            self.thread = threading.Thread(target=loop, daemon=True)
            self.thread.start()
            t = time.perf_counter()
            while not self.samples and time.perf_counter() - t < 5.0:
                time.sleep(0.002)
            return
        except Exception:
            self.thread = None
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.proc = None

    def mark_start(self):
        self.t0 = time.perf_counter()

    def mark_stop(self):
        self.t1 = time.perf_counter()

    def stop(self):
        if self.thread is not None:
            time.sleep(0.01)
            self.stop_flag.set()
            self.thread.join(timeout=2)
            t0 = self.t0 if self.t0 is not None else -1e30
            t1 = self.t1 if self.t1 is not None else 1e30
            inside = [x for x in self.samples if t0 <= x[0] <= t1]
            # a region shorter than the poll period: the samples bracketing it
            use = inside or [x for x in self.samples if x[0] <= t0][-1:] + \
                [x for x in self.samples if x[0] >= t1][:1]
            reasons = sorted(nm for nm, b in self.bits.items() if any(x[2] & b for x in use))
            return {"sm_mhz": statistics.median(x[1] for x in use) if use else None,
                    "sm_max_mhz": self.max_mhz, "samples": len(use),
                    "samples_in_timed_region": len(inside), "source": "nvml, 2 ms poll",
                    "reasons": reasons}
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:  # pragma: no cover
            self.proc.kill()
        sms, maxs, reasons = [], [], set()
        for line in Path(self.path).read_text().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sms.append(float(parts[1]))
                maxs.append(float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(self.NAMES, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        os.unlink(self.path)
        return {"sm_mhz": statistics.median(sms) if sms else None,
                "sm_max_mhz": max(maxs) if maxs else None, "samples": len(sms),
                "source": "nvidia-smi -lms 100", "reasons": sorted(reasons)}


def measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def host_link_peak(dev, nbytes=512 << 20, reps=10):
    """Measured host -> device rate of this box's link: a pinned host buffer
    copied into HBM by the copy engine (best of ``reps``, CUDA events).  The
    host-store gather reads the same pinned memory over the same link with
    SM loads, so this is its ceiling."""
    import torch

    src = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    dst = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    best = None
    for _ in range(reps + 1):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        dst.copy_(src, non_blocking=True)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b)
        best = ms if best is None else min(best, ms)
    del src, dst
    return nbytes / (best * 1e-3) / 1e9


def traffic_table():
    """Per-launch DRAM bytes of each kernel from the committed ncu capture."""
    files = sorted((ROOT / "profiles").glob("traffic_*.json"))
    if not files:
        return {}
    return json.loads(files[-1].read_text())


# ------------------------------------------------------------------- arms
def run_reference_arm(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return 0
    import torch
    device = "cuda" if torch.cuda.is_available() else None
    sg, fanouts, t_gen = build_inputs(args, device)
    ro, col, feats, labels = host_arrays(sg)
    mask = oracle_cache_mask(ro, col, np.asarray(sg.train_mask), args.cache_fraction, args.seed,
                             fanouts)
    from paper_2601_04707_b200.runtime import epoch_permutation
    perm = epoch_permutation(np.asarray(sg.train_mask), args.seed, 0)
    del sg
    if device:
        torch.cuda.empty_cache()
    # warm-up batches (W of them, as the driver asked; a cap far above any
    # driver W keeps a mistaken W from running for hours) are not timed; each
    # timed step is one batch, capped so the whole arm stays within minutes
    w = min(args.warmup, 64)
    cpu_oracle_run(ro, col, feats, labels, mask, perm, fanouts, args, 60.0, w, workers=1)
    budget = float(os.environ.get("MQ_REF_BUDGET_S", 90.0))
    seeds, nb, dt, cores = cpu_oracle_run(ro, col, feats, labels, mask, perm[w * args.batch:],
                                          fanouts, args, budget, args.steps + 1, bid0=w)
    value = seeds / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": nb, "warmup": w, "ms_per_step": dt * 1e3 / max(nb, 1),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic", "config": {"workload": SHAPE_DESC[args.shape],
                                        "parallelism": "cpu oracle, rank 0 only"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": f"{nb} batches x {args.batch} seeds of the {args.shape} "
                                   f"workload (oracle/ NumPy restatement of mqpipe, pinned to "
                                   f"reference golden vectors; {cores - 1} sampler processes + "
                                   f"1 compute process), {dt:.1f} s steady state (pool "
                                   f"start-up and the first batch not timed)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def spawn_ranks(args):
    """`bench.py --gpus N` without a launcher: start N ranks, one per GPU, with
    the torchrun environment (RANK / LOCAL_RANK / WORLD_SIZE / MASTER_*)."""
    import torch
    import torch.multiprocessing as mp
    share = os.environ.get("MQ_DIST_BACKEND") == "gloo"
    if not share and torch.cuda.device_count() < args.gpus:
        print(json.dumps({"error": f"--gpus {args.gpus} but {torch.cuda.device_count()} CUDA "
                                   f"device(s) visible (MQ_DIST_BACKEND=gloo shares one GPU "
                                   f"for a functional run)"}), flush=True)
        return 2
    import socket
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    mp.start_processes(_spawned_rank, args=(args, port), nprocs=args.gpus, join=True,
                       start_method="spawn")
    return 0


def _spawned_rank(rank, args, port):
    os.environ.update(RANK=str(rank), LOCAL_RANK=str(rank), WORLD_SIZE=str(args.gpus),
                      MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    if args.impl == "reference":
        run_reference_arm(args)
    else:
        run_ours(args)


def run_ours(args):
    import torch
    import torch.distributed as dist
    rank, world, local = env_rank()
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    # one GPU per rank; MQ_DIST_BACKEND=gloo lets ranks share GPUs (a
    # functional multi-rank check on a single-GPU box, not a perf setup)
    share = os.environ.get("MQ_DIST_BACKEND") == "gloo"
    if not share and world > torch.cuda.device_count():
        raise SystemExit(f"{world} ranks but {torch.cuda.device_count()} GPUs")
    local = local % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        # host plumbing only (handle exchange, barriers, the max over ranks):
        # the data path is the peer-memory exchange inside the step graphs
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    import paper_2601_04707_b200 as mq
    from paper_2601_04707_b200._lib import lib
    from paper_2601_04707_b200.runtime import epoch_permutation

    setup = {}
    sharded = args.feature_placement == "sharded"
    sg, fanouts, setup["graph_gen_s"] = build_inputs(
        args, f"cuda:{local}", feature_shard=(world, rank) if sharded else None)
    t0 = time.perf_counter()
    g = mq.DeviceGraph.from_csr(sg, device=dev, feature_placement=args.feature_placement)
    torch.cuda.synchronize()
    setup["upload_s"] = time.perf_counter() - t0
    if args.shape == "papers" or sharded:  # no host copy of the features for the CPU leg
        args.no_cpu_baseline = True
    if args.no_cpu_baseline:  # the generator's device arrays are not needed any more
        sg.col_indices = sg.row_offsets = sg.labels = None
        if sg.features is not g.features:
            sg.features = None
        torch.cuda.empty_cache()
    # per-epoch GNS residency on the device (refresh_cache under the refresh
    # injected-draw contract; degree mode when most nodes train, else walk —
    # the reference driver's choose_cache_mode, bench.py:65-72)
    cache_mode = "degree" if float(np.mean(g.train_mask)) >= 0.5 else "walk"

    def refresh(epoch):
        probs = (mq.cache_probs_degree(g) if cache_mode == "degree"
                 else mq.cache_probs_walk(g, fanouts[0], len(fanouts)))
        return mq.refresh_cache(g, probs, args.cache_fraction, mq.RefreshStream(args.seed, epoch))

    t0 = time.perf_counter()
    cache = refresh(0)
    torch.cuda.synchronize()
    setup["cache_refresh_s"] = time.perf_counter() - t0
    mask = cache.cached_mask.cpu().numpy()
    model = mq.init_model(g.feature_dim, args.hidden, g.num_classes, num_layers=len(fanouts),
                          seed=args.seed, learning_rate=1e-3, device=dev)
    n_train = int(g.train_mask.sum())
    windows = -(-n_train // (args.batch * world))
    if args.no_pdl:
        lib().mq_set_pdl(0)
    if os.environ.get("MQ_TC_GRID_CAP"):
        lib().mq_set_tc_grid_cap(int(os.environ["MQ_TC_GRID_CAP"]))
    if os.environ.get("MQ_TC_KERNEL"):  # A/B of the tcgen05 GEMM kernels (mqgnn.h)
        lib().mq_set_tc_kernel(int(os.environ["MQ_TC_KERNEL"]))
    queue_choice = None
    if args.queue_depth == "auto":  # the reference's --queue auto (autotune.py), measured
        from paper_2601_04707_b200.autotune import auto_queue_depth
        queue_choice = auto_queue_depth(g, model, fanouts=fanouts, batch_size=args.batch,
                                        num_train=n_train, cache=cache, seed=args.seed)
        args.queue_depth = queue_choice.depth
    elif args.queue_depth is not None:
        args.queue_depth = int(args.queue_depth)
    fx, exchange_kind = None, None
    if world > 1:
        peer_ok = args.exchange == "peer" and (share or all(
            torch.cuda.can_device_access_peer(local, q) for q in range(world) if q != local))
        if peer_ok:  # RaCoM publish/apply over NVLink peer memory, inside the graphs
            fx = mq.PeerExchange(model.dev.num_params, dev, lag=args.staleness, ring=4)
            exchange_kind = f"peer memory (NVLink P2P), staleness {args.staleness}"
        else:
            exchange_kind = "torch.distributed all_reduce (f64), host-issued"
    runner = mq.StepRunner(g, model, fanouts=fanouts, batch_size=args.batch, num_train=n_train,
                           cache=cache, optimizer="adam", seed=args.seed, world=world, rank=rank,
                           multi=world > 1, queue_depth=args.queue_depth,
                           pipeline=not args.no_pipeline, layer0=args.layer0, exchange=fx)
    exchange = mq.DistExchange() if world > 1 else None
    driver = mq.WindowDriver([runner], exchange, sync_period=1)
    t0 = time.perf_counter()
    runner.capture()
    setup["capture_s"] = time.perf_counter() - t0
    epoch = [0]
    runner.begin_epoch(0, epoch_permutation(g.train_mask, args.seed, 0))
    seeds_done = [0]
    plan_sizes = np.minimum(args.batch, np.maximum(
        0, n_train - np.arange(windows * world) * args.batch))

    # MQ_BENCH_EPOCH_TIMES=1: train-stream events at every epoch boundary
    # (diagnostic; the per-epoch device times go to stderr)
    epoch_evs = [] if os.environ.get("MQ_BENCH_EPOCH_TIMES") else None

    def run_windows(n):
        """n windows; a single replica issues whole slot groups as one graph each."""
        left = n
        while left > 0:
            if runner.windows_done >= windows:
                if epoch_evs is not None:
                    epoch_evs.append(torch.cuda.Event(enable_timing=True))
                    epoch_evs[-1].record(runner.stream)
                runner.finish()  # a lagged exchange applies its held-back window
                epoch[0] += 1
                runner.begin_epoch(epoch[0], epoch_permutation(g.train_mask, args.seed, epoch[0]))
            k = runner.windows_done
            if world == 1 or fx is not None:  # whole slot groups as one graph each
                done = runner.steps(left, windows)
            else:  # replicas start identical (same init) and apply the same
                # all-reduced window, so the per-window model average is the
                # identity (WindowDriver's exact sync elision) and is not issued
                runner.compute_window()
                driver._reduce([runner.grad64])
                runner.apply_window()
                done = 1
            for kk in range(k, k + done):
                for r in range(world):
                    seeds_done[0] += int(plan_sizes[kk * world + r])
            left -= done

    run_windows(args.warmup)
    # the timed region starts at a slot-group boundary, so every timed window
    # runs inside a group graph (whole groups, and an epoch's or the run's
    # last k < Q windows as one partial-group graph) instead of a mix of
    # group and single-window graphs; W stays a minimum
    extra_warm = 0
    if world == 1 and runner.pipeline:
        extra_warm = (-runner.windows_done) % runner.Q
        run_windows(extra_warm)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.05)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    seeds_done[0] = 0
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    # a ~1 ms device spin ahead of ev0 lets the host enqueue the first graph
    # launches before the timed region opens: the K timed steps are then
    # device time only, not the host's first-launch latency (which a short
    # run would otherwise carry, ~6 us/step at K = 20)
    with torch.cuda.stream(runner.stream):
        torch.cuda._sleep(2_000_000)
    clocks.mark_start()
    ev0.record(runner.stream)
    t_wall = time.perf_counter()
    run_windows(args.steps)
    ev1.record(runner.stream)
    torch.cuda.synchronize()
    t_wall = time.perf_counter() - t_wall
    clocks.mark_stop()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    ms = ev0.elapsed_time(ev1)
    if epoch_evs:
        marks = [e for e in epoch_evs if e.query()]
        print(json.dumps({"epoch_ms": [round(a.elapsed_time(b), 3)
                                       for a, b in zip(marks, marks[1:])]}), file=sys.stderr)
    ms_t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_max = float(ms_t.item())
    runner.check_finite()
    value = seeds_done[0] / (ms_max / 1e3)

    # -------- per-kernel profile: each op replayed in a CUDA graph, warm --------
    per_kernel = {}
    n_kernels = runner.kernels_per_step()
    if rank == 0 and args.profile_steps > 0:
        from paper_2601_04707_b200.profiling import op_table
        tab = op_table(runner, reps=args.profile_steps)
        Q = runner.Q
        per_step = {nm: rec["us"] * (1.0 / Q if nm.startswith("prep_") else 1.0)
                    for nm, rec in tab["ops"].items()}
        tot = sum(per_step.values())
        for nm, rec in tab["ops"].items():
            per_kernel[nm] = {
                "avg_launch_us": rec["us"], "us_per_step": per_step[nm],
                "share": per_step[nm] / tot, "units": rec.get("units"),
                "bytes_per_launch": rec.get("bytes"), "gbps": rec.get("gbps"),
                "flops_per_launch": rec.get("flops"), "tflops": rec.get("tflops"),
                "sector_gbps": rec.get("sector_gbps"),
            }
        per_kernel["_counts"] = tab["counts"]
    # ---- host-miss gather against the host link (configs[3]: features in
    # pinned host memory, only the GNS cache table in HBM): the misses of
    # one prep pass cross the link inside prep_gather
    host_link = None
    if rank == 0 and args.feature_placement == "host" and "prep_gather" in per_kernel:
        hr = cache.hit_rate()
        n_in = int(per_kernel["_counts"]["hops"][-1][1])
        miss_bytes = (1.0 - hr) * runner.Q * n_in * 4 * g.feature_dim
        us = per_kernel["prep_gather"]["avg_launch_us"]
        peak = host_link_peak(dev)
        ach = miss_bytes / (us * 1e-6) / 1e9
        host_link = {"bound": "host link", "achieved": ach, "peak": peak, "unit": "GB/s",
                     "frac": ach / peak, "miss_rate": 1.0 - hr,
                     "miss_bytes_per_pass": miss_bytes, "prep_gather_us": us,
                     "units": f"{runner.Q} batches x {n_in} input rows x {g.feature_dim} f32",
                     "peak_source": "measured: 512 MiB pinned host -> HBM copy_, best of 10, "
                                    "CUDA events (copy engine; the gather reads the link "
                                    "with SM loads and can exceed it)"}
    if world > 1:  # the other ranks' next steps wait on rank 0's exchange
        dist.barrier()
    # ----------------------------- e2e through the host-buffer entry point ---
    e2e = None
    if world == 1 or fx is not None:
        if fx is not None:  # epoch boundary: nothing held back by a lagged exchange
            runner.finish()
        runner.capture_host_input()
        B = args.batch
        # the round-robin deal (runtime.py:111-113): this rank's batches j = rank, rank + N, ...
        # over as many fresh epoch permutations as --e2e-steps needs (distinct
        # targets and batch ids throughout: one epoch of the Reddit shape is
        # only ~150 windows, too short to amortise the first group's prep)
        host_batches, ep = [], 100
        while len(host_batches) < args.e2e_steps:
            perm_e2e = epoch_permutation(g.train_mask, args.seed, ep)
            per = len(perm_e2e) // (B * world)
            if per == 0:
                break
            for j in range(min(per, args.e2e_steps - len(host_batches))):
                host_batches.append((len(host_batches) * world + rank, torch.from_numpy(
                    perm_e2e[(j * world + rank) * B:(j * world + rank + 1) * B]
                    .astype(np.int32)).pin_memory()))
            ep += 1
        nb = len(host_batches)
        for _ in runner.run_host_batches(host_batches[:5]):
            pass
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0.record(runner.stream)
        seeds = 0
        for _bid, _loss in runner.run_host_batches(host_batches):
            pass
        seeds = sum(int(t.numel()) for _, t in host_batches) * world
        e1.record(runner.stream)
        torch.cuda.synchronize()
        e2e_ms = e0.elapsed_time(e1)
        if world > 1:
            t = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_ms = float(t.item())
        e2e = {"value": seeds / (e2e_ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": 4 * B + 16,
               "d2h_bytes_per_step": 8, "steps": nb, "ms_per_step": e2e_ms / nb,
               "entry": "StepRunner.run_host_batches (per batch: pinned targets H2D, graph, loss D2H)"}
    runner.check_finite()

    # ----------------------------------------------------------- CPU baseline
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        ro, col, feats, labels = host_arrays(sg)
        perm = epoch_permutation(g.train_mask, args.seed, 0)
        seeds, nbat, dt, cores = cpu_oracle_run(ro, col, feats, labels, mask, perm, fanouts, args,
                                                args.cpu_seconds, 10_000)
        cpu = {"value": seeds / dt, "unit": UNIT, "cores": cores, "kind": "port",
               "sample": f"{nbat} batches x {args.batch} seeds of the same workload through the "
                         f"oracle (NumPy restatement of mqpipe's per-batch path; {cores - 1} "
                         f"sampler processes + 1 compute process), {dt:.1f} s steady state "
                         f"(pool start-up and the first batch not timed)"}

    # ------------------------------ per-epoch work outside the timed steps
    epoch_extra = None
    if rank == 0 and world == 1:
        def ev_ms(fn, reps=2):
            fn()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(reps):
                fn()
            b.record()
            torch.cuda.synchronize()
            return a.elapsed_time(b) / reps
        acc = [0.0]

        def ev():
            acc[0] = mq.evaluate(g, model, g.val_mask)
        try:
            epoch_extra = {"cache_mode": cache_mode,
                           "refresh_ms": ev_ms(lambda: refresh(1)),
                           "evaluate_ms": ev_ms(ev),
                           "val_acc_after_timed_steps": acc[0],
                           "val_nodes": int(np.count_nonzero(g.val_mask)),
                           "note": "per-epoch device work (refresh_cache + full-graph evaluate), "
                                   "CUDA-event timed; not part of epoch_ms (training only)"}
        except (torch.OutOfMemoryError, RuntimeError) as exc:  # report, keep the bench line
            epoch_extra = {"cache_mode": cache_mode, "error": str(exc).splitlines()[0][:200]}
            torch.cuda.empty_cache()
    if rank == 0:
        hbm, peak_kind = measured_peaks()
        kern = {k: v for k, v in per_kernel.items() if not k.startswith("_")}
        # the dominant kernel of the step's critical path: the train stream (the
        # prep_* ops run concurrently on the prep stream, one pass per Q windows)
        crit = {k: v for k, v in kern.items() if not k.startswith("prep_")}
        dom = max(crit.items(), key=lambda kv: kv[1]["us_per_step"]) if crit else None
        traffic = traffic_table()
        roof = None
        if dom:
            name, kd = dom
            achieved = kd["gbps"]
            roof = {"kernel": name, "bound": "hbm", "achieved": achieved, "peak": hbm,
                    "unit": "GB/s", "frac": (achieved / hbm) if achieved else None,
                    "traffic": traffic.get(name), "peak_source":
                        f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs)",
                    "algorithmic_bytes_per_launch": kd["bytes_per_launch"],
                    "avg_launch_us": kd["avg_launch_us"], "share_of_step": kd["share"],
                    "timing": "CUDA-event time of the op replayed 20x in a CUDA graph (no PDL) "
                              "(warm, same buffers as the step)",
                    "choice": "largest share of the train-stream critical path"}
            if kd.get("tflops"):
                roof["tflops_fp32_equiv"] = kd["tflops"]
        focus = {}
        for nm in ("prep_sample", "prep_relabel", "prep_gather", "prep_pass", "sage_aggregate_l0",
                   "sage_head", "sage_transform_l0", "sage_transform_bwd_l0",
                   "sage_scatter_bwd_l0", "optimizer"):
            if nm in kern:
                k = kern[nm]
                focus[nm] = {"gbps": k["gbps"], "frac_hbm": (k["gbps"] / hbm if k["gbps"] else None),
                             "avg_launch_us": k["avg_launch_us"], "share": k["share"],
                             "units": k["units"]}
                if k.get("tflops"):
                    focus[nm]["tflops_fp32_equiv"] = k["tflops"]
                if k.get("sector_gbps"):  # random-access kernels: 32 B per touch
                    focus[nm]["sector_gbps"] = k["sector_gbps"]
                    focus[nm]["frac_hbm_sector"] = k["sector_gbps"] / hbm
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "warmup_windows_run": args.warmup + extra_warm,
            "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (Chung-Lu power law, exponent 2.1, N(0,1) features, teacher "
                    "labels; random-init weights)",
            "config": {"workload": SHAPE_DESC[args.shape], "nodes": g.num_nodes,
                       "arcs": g.num_edges, "feature_dim": g.feature_dim,
                       "classes": g.num_classes, "fanouts": list(fanouts), "batch": args.batch,
                       "hidden": args.hidden, "cache_fraction": args.cache_fraction,
                       "optimizer": "adam", "feature_placement": args.feature_placement,
                       "parallelism": f"dp{world} (RaCoM sync P=1)" if world > 1 else "dp1",
                       "exchange": exchange_kind,
                       "l2": "inputs larger than L2 (CSR+features ~1.1 GB), no flush",
                       "cuda_graph": True, "queue_depth": runner.Q,
                       "pdl": bool(lib().mq_get_pdl()), "pipeline": runner.pipeline,
                       "queue_auto": None if queue_choice is None else {
                           "cap": queue_choice.cap, "formula_eq24": queue_choice.formula_depth,
                           "ms_per_window": queue_choice.ms_per_window},
                       "layer0": "aggregate-first" if getattr(runner.tw, "af0", False)
                                 else "transform-first"},
            "epoch_ms": ms_max / args.steps * windows, "windows_per_epoch": windows,
            "roofline": roof, "kernels": focus,
            "cpu_baseline": cpu, "e2e": e2e, "clocks": clk, "per_epoch": epoch_extra,
            "cache": {"mode": cache_mode, "fraction": args.cache_fraction,
                      "resident": cache.size, "hit_rate": cache.hit_rate()},
            "host_link": host_link,
            "gpu_launches": int(round(n_kernels * args.steps)), "kernels_per_step": n_kernels,
            "wall_s_timed": t_wall, "setup": setup,
        }
        print(json.dumps(line), flush=True)
        if os.environ.get("MQ_BENCH_KERNELS"):
            print(json.dumps({"per_kernel": per_kernel}), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:  # no launcher: spawn the ranks
        return spawn_ranks(args)
    if args.impl == "reference":
        return run_reference_arm(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
