"""GPU: the runner's side streams are ordered after the caller's stream.

Buffers, weights and caches are created (zero-filled, copied) on the caller's
current stream while the step graphs run on the runner's own streams.  A
regression test for the race compute-sanitizer racecheck exposed (the
device permutation's zero-fill landing after the epoch's permutation copy,
so the first prep pass cut wrong targets): the default stream is kept busy
with a long sleep kernel while the runner is built and its first batch
prepared; the batch must still be the planned one.
"""

import numpy as np
import pytest

from conftest import load_golden, make_g2

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2601_04707_b200 as mq  # noqa: E402
from paper_2601_04707_b200.runtime import epoch_permutation  # noqa: E402


def test_first_prep_sees_initialised_buffers():
    gs = load_golden("sampling.npz")
    hg = make_g2(gs)
    g = mq.DeviceGraph.from_csr(hg)
    torch.cuda.synchronize()
    torch.cuda._sleep(200_000_000)  # ~0.1 s of work queued on the default stream
    state = mq.init_model(16, 16, 5, num_layers=2, seed=7, learning_rate=0.01)
    perm = epoch_permutation(hg.train_mask, 5, 0)
    r = mq.StepRunner(g, state, fanouts=(4, 3), batch_size=64, num_train=perm.size, seed=5,
                      use_graph=False, pipeline=False)
    r.begin_epoch(0, perm)
    sw = r.groups[0].slots[0]
    with torch.cuda.stream(r.stream):
        r._enqueue_prep(sw, r.stream.cuda_stream)
    torch.cuda.synchronize()
    assert np.array_equal(sw.targets[:64].cpu().numpy(), perm[:64])
