import sys
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import torch
from conftest import load_golden, make_g2
import paper_2601_04707_b200 as mq
from paper_2601_04707_b200._lib import lib
gs = load_golden("sampling.npz")
hg = make_g2(gs)
pdl = int(sys.argv[1]) if len(sys.argv) > 1 else 1
lib().mq_set_pdl(pdl)
layer0 = sys.argv[2] if len(sys.argv) > 2 else "auto"
g = mq.DeviceGraph.from_csr(hg)
cache = mq.DeviceCache(g, gs["g2/mask10"])
st = mq.init_model(16, 16, 5, num_layers=2, seed=5, learning_rate=0.01)
from paper_2601_04707_b200.runtime import epoch_permutation
perm = epoch_permutation(hg.train_mask, 5, 0)
r = mq.StepRunner(g, st, fanouts=(4, 3), batch_size=64, num_train=perm.size, cache=cache, seed=5, layer0=layer0)
try:
    r.capture()
    print("pdl", pdl, layer0, "capture OK", r.launches_per_phase)
except Exception as e:
    print("pdl", pdl, layer0, "FAILED", type(e).__name__, str(e)[:300])
    print("last error:", lib().mq_last_error())
