"""RaCoM over peer memory: gradient sharing with no collective on the data path.

Reference: ``mqpipe/racom.py:36-87`` (Accumulator, apply_update),
``racom.py:142-184`` (share_gradient broadcasts every packet to every
device), ``runtime.py:167-195`` (windows applied in order).

Every rank owns an arena (``mq_peer_alloc``) that the other ranks map through
CUDA IPC (NVLink P2P between GPUs; the same physical pages for ranks that
share a GPU).  Per window the train stream runs

    ... backward -> mq_racom_publish -> mq_racom_apply

``publish`` writes the rank's f32 packet into its own arena and raises its
flag word in every arena; ``apply`` waits on the local flag words, folds the
ranks' packets in rank order into the reference's f64 running mean and runs
the optimizer.  Both are ordinary stream-ordered kernels, so a multi-rank
window is one CUDA-graph replay like a single-GPU window.  ``lag = 1`` gives
the pipelined schedule (window k applied after window k+1's backward:
staleness exactly 1); ``lag = 0`` the reference's serial parity
schedule.

Handles travel over ``torch.distributed`` (any backend: host plumbing only).
In-process replicas (the reference's simulated devices sharing one process)
alias the arenas directly.
"""

from __future__ import annotations

import ctypes as C
import os

import torch

from ._lib import I32, I64, P, lib, ptr

MQ_MAX_PEERS = 8
PEER_HEADER_BYTES = 256


class IpcHandle(C.Structure):
    _fields_ = [("bytes", C.c_ubyte * 64)]


class PeerDesc(C.Structure):
    """mq_peer_exchange (include/mqgnn.h)."""
    _fields_ = [("world", I32), ("rank", I32), ("ring", I32), ("pad_", I32),
                ("n", I64), ("timeout_ns", I64), ("arena", P * MQ_MAX_PEERS)]


class PeerArena:
    """One cudaMalloc'd, zeroed device buffer exportable to other processes."""

    def __init__(self, nbytes: int, device):
        self.device = torch.device(device)
        self.nbytes = int(nbytes)
        out = C.c_void_p()
        with torch.cuda.device(self.device):
            lib().mq_peer_alloc(self.nbytes, C.byref(out))
        self.ptr = int(out.value)

    def export(self) -> bytes:
        h = IpcHandle()
        with torch.cuda.device(self.device):
            lib().mq_ipc_export(self.ptr, C.byref(h))
        return C.string_at(C.addressof(h), C.sizeof(h))  # all 64 bytes (NULs included)

    def free(self):
        if self.ptr:
            with torch.cuda.device(self.device):
                lib().mq_peer_free(self.ptr)
            self.ptr = 0


def open_handle(handle: bytes, device) -> int:
    if len(handle) != C.sizeof(IpcHandle):
        raise ValueError("malformed IPC handle")
    h = IpcHandle()
    C.memmove(C.addressof(h), handle, len(handle))
    out = C.c_void_p()
    with torch.cuda.device(torch.device(device)):
        lib().mq_ipc_open(C.byref(h), C.byref(out))
    return int(out.value)


def exchange_handles(local: bytes, group=None):
    """all-gather of (pid, device uuid, handle) over torch.distributed."""
    import torch.distributed as dist
    me = (os.getpid(), local)
    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, me, group=group)
    return out


class PeerExchange:
    """The fused RaCoM exchange of one rank (``fused_exchange`` for
    ``trainer.StepRunner``).  ``world``/``rank`` come from torch.distributed
    unless ``local_arenas`` (in-process replicas) is given."""

    fused = True

    def __init__(self, num_params: int, device, *, ring: int = 4, lag: int = 0,
                 timeout_s: float = 30.0, group=None, local_arenas=None, rank: int | None = None):
        if lag not in (0, 1):
            raise ValueError("lag must be 0 (parity schedule) or 1 (pipelined, staleness 1)")
        if ring < lag + 2:
            raise ValueError("ring must exceed lag + 1")
        self.device = torch.device(device)
        self.n = int(num_params)
        self.ring = int(ring)
        self.lag = int(lag)
        self._opened = []
        self.owns = None
        nbytes = int(lib().mq_peer_arena_bytes(self.n, self.ring))
        if local_arenas is not None:  # replicas of this process share the arenas
            self.world, self.rank = len(local_arenas), int(rank)
            ptrs = [a.ptr for a in local_arenas]
        else:
            import torch.distributed as dist
            self.world, self.rank = dist.get_world_size(group), dist.get_rank(group)
            if self.world > MQ_MAX_PEERS:
                raise ValueError(f"at most {MQ_MAX_PEERS} ranks share gradients over peer memory")
            self.owns = PeerArena(nbytes, self.device)
            torch.cuda.synchronize(self.device)
            infos = exchange_handles(self.owns.export(), group)
            ptrs = []
            for q, (pid, h) in enumerate(infos):
                if q == self.rank:
                    ptrs.append(self.owns.ptr)
                elif pid == os.getpid():
                    raise RuntimeError("two ranks in one process: pass local_arenas")
                else:
                    p = open_handle(h, self.device)
                    self._opened.append(p)
                    ptrs.append(p)
            torch.cuda.synchronize(self.device)
            dist.barrier(group)  # every arena is mapped before anyone publishes
        d = PeerDesc()
        d.world, d.rank, d.ring = self.world, self.rank, self.ring
        d.n = self.n
        d.timeout_ns = int(timeout_s * 1e9)
        for q, p in enumerate(ptrs):
            d.arena[q] = p
        self.desc = d

    @staticmethod
    def local_group(num_params: int, device, world: int, **kw):
        """Exchanges for ``world`` replicas living in this process."""
        ring = kw.get("ring", 4)
        nbytes = int(lib().mq_peer_arena_bytes(int(num_params), int(ring)))
        arenas = [PeerArena(nbytes, device) for _ in range(world)]
        exs = [PeerExchange(num_params, device, local_arenas=arenas, rank=r, **kw)
               for r in range(world)]
        exs[0]._keep = arenas
        return exs

    # ----------------------------------------------------------- launches
    def publish(self, grad32: torch.Tensor, src, n_targets: torch.Tensor, stream: int):
        lib().mq_racom_publish(C.byref(self.desc), ptr(grad32),
                               C.byref(src) if src is not None else None, ptr(n_targets), stream)

    def apply(self, model, optimizer: str, stream: int, lag: int | None = None):
        opt = {"adam": 0, "sgd": 1}[optimizer]
        lib().mq_racom_apply(C.byref(self.desc), opt, self.lag if lag is None else int(lag),
                             ptr(model.flat_w), ptr(model.flat_m), ptr(model.flat_v),
                             ptr(model.step_dev), ptr(model.bias), model.bias_len,
                             ptr(model.lr_dev), ptr(model.nonfinite), stream)

    def state(self, stream=None) -> dict:
        out = torch.zeros(4, dtype=torch.int64, device=self.device)
        s = stream if stream is not None else torch.cuda.current_stream(self.device).cuda_stream
        lib().mq_peer_state(C.byref(self.desc), ptr(out), s)
        pub, app, lo, hi = out.cpu().tolist()
        return {"published": pub, "applied": app, "min_flag": lo, "max_flag": hi}

    def close(self):
        for p in self._opened:
            lib().mq_ipc_close(p)
        self._opened = []
        if self.owns is not None:
            self.owns.free()
            self.owns = None
