"""Diagnostic: 2 ranks (gloo, shared GPU) over the in-graph peer exchange:
per-window losses of one epoch through step() vs steps(full) vs steps(5/4)."""
import os
import socket
import sys
from pathlib import Path

import numpy as np
import torch
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def worker(rank, world, port, modes):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    import torch.distributed as dist
    import paper_2601_04707_b200 as mq
    from conftest import load_golden, make_g2
    from paper_2601_04707_b200.graph import DeviceGraph
    from paper_2601_04707_b200.runtime import epoch_permutation
    dist.init_process_group("gloo", rank=rank, world_size=world)
    gs = load_golden("sampling.npz")
    hg = make_g2(gs)
    g = DeviceGraph.from_csr(hg)
    cache = mq.DeviceCache(g, gs["g2/mask10"])
    B = 64
    perm = epoch_permutation(hg.train_mask, 5, 0)
    windows = -(-perm.size // (B * world))
    for mode in modes:
        st = mq.init_model(16, 16, 5, num_layers=2, seed=5, learning_rate=0.01)
        fx = mq.PeerExchange(st.dev.num_params, g.device, lag=0, ring=4)
        r = mq.StepRunner(g, st, fanouts=(4, 3), batch_size=B, num_train=perm.size, cache=cache,
                          seed=5, world=world, rank=rank, multi=True, queue_depth=3, exchange=fx,
                          use_graph=mode != "eager")
        r.begin_epoch(0, perm)
        if mode != "eager":
            r.capture()
        done, c = 0, 0
        while done < windows:
            if mode == "full":
                done += r.steps(windows, windows)
            elif mode == "chunked":
                done += r.steps(5 if c % 2 == 0 else 4, windows)
            else:
                r.step()
                done += 1
            c += 1
        r.finish()
        l = r.losses(windows)
        torch.cuda.synchronize()
        dist.barrier()
        fx.close()
        print(f"rank {rank} {mode:8s}", np.array2string(l[:6], precision=5), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    modes = sys.argv[1:] or ["windows", "full", "chunked", "eager"]
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    mp.start_processes(worker, args=(2, port, modes), nprocs=2, join=True, start_method="spawn")
