import sys
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np
import torch
from conftest import load_golden, make_g2
import paper_2601_04707_b200 as mq
from paper_2601_04707_b200._lib import lib
gs = load_golden("sampling.npz")
hg = make_g2(gs)
g = mq.DeviceGraph.from_csr(hg)
cache = mq.DeviceCache(g, gs["g2/mask10"])
def run(fused, use_graph=True, pipeline=True, pdl=1):
    lib().mq_set_pdl(pdl)
    cfg = mq.PipelineConfig(num_devices=1, batch_size=64, sampler=mq.SamplerParams("sage", (4, 3), num_layers=2),
                            optimizer="adam", seed=5, fused_step=fused, use_graph=use_graph, pipeline=pipeline)
    st = mq.init_model(16, 16, 5, num_layers=2, seed=5, learning_rate=0.01)
    stats, _ = mq.run_epoch(g, cache, [st], cfg, epoch=0)
    return np.array([stats.losses[b] for b in sorted(stats.losses)])
ref = run(False)
for args in [dict(fused=True), dict(fused=True, pdl=0), dict(fused=True, use_graph=False), dict(fused=True, pipeline=False), dict(fused=True, use_graph=False, pipeline=False)]:
    l = run(**args)
    print(args, "max rel", float(np.max(np.abs(l - ref) / np.abs(ref))), l[:4], ref[:4])
