import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = Path(__file__).resolve().parent / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libmqgnn.so")
    config.addinivalue_line("markers", "slow: long-running (full-size shapes)")


def load_golden(name):
    return dict(np.load(GOLDEN / name, allow_pickle=False))


@pytest.fixture(scope="session")
def golden_sampling():
    return load_golden("sampling.npz")


@pytest.fixture(scope="session")
def golden_nn():
    return load_golden("nn.npz")


@pytest.fixture(scope="session")
def golden_cache():
    return load_golden("cache.npz")


@pytest.fixture(scope="session")
def golden_runtime():
    return load_golden("runtime.npz")


EDGES_8 = [
    (0, 1), (1, 0), (0, 2), (2, 0), (1, 2), (2, 1),
    (2, 3), (3, 2), (3, 3), (3, 4), (4, 3), (4, 5), (5, 4),
    (5, 6), (6, 5), (6, 7), (7, 6), (7, 0), (0, 7),
    (1, 5), (5, 1), (2, 6), (6, 2),
]


class HostGraph:
    """Minimal GraphCSR-like container for tests (graph.py:28-91 fields)."""

    def __init__(self, row_offsets, col_indices, features, labels, num_classes,
                 train_mask=None):
        self.num_nodes = len(row_offsets) - 1
        self.row_offsets = np.asarray(row_offsets, dtype=np.int64)
        self.col_indices = np.asarray(col_indices, dtype=np.int64)
        self.features = np.asarray(features, dtype=np.float32)
        self.labels = np.asarray(labels, dtype=np.int32)
        self.num_classes = num_classes
        n = self.num_nodes
        self.train_mask = (np.zeros(n, bool) if train_mask is None
                           else np.asarray(train_mask, bool))
        self.val_mask = np.zeros(n, bool)
        self.test_mask = np.zeros(n, bool)

    @property
    def feature_dim(self):
        return self.features.shape[1]

    @property
    def num_edges(self):
        return self.col_indices.size


def csr_from_edges(edges, n):
    e = np.asarray(edges, dtype=np.int64).reshape(-1, 2)
    keys = np.unique(e[:, 0] * n + e[:, 1])
    src, dst = keys // n, keys % n
    ro = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(src, minlength=n), out=ro[1:])
    return ro, dst


def make_g8():
    rng = np.random.default_rng(42)
    feats = rng.standard_normal((8, 3)).astype(np.float32)
    labels = np.array([0, 1, 0, 1, 0, 1, 0, 1], dtype=np.int32)
    ro, col = csr_from_edges(EDGES_8, 8)
    return HostGraph(ro, col, feats, labels, 2)


def make_g2(golden):
    return HostGraph(golden["g2/row_offsets"], golden["g2/col_indices"], golden["g2/features"],
                     golden["g2/labels"], 5, golden["g2/train_mask"])


def make_cfg1():
    from paper_2601_04707_b200.synth import generate_numpy
    sg = generate_numpy(10_000, 100_000, 64, 4, train=0.66, seed=0)
    return HostGraph(sg.row_offsets, sg.col_indices, sg.features, sg.labels, 4, sg.train_mask)


def golden_batch(golden, prefix):
    """(targets, layers[list of dict], digest hex, hits) of a stored batch."""
    layers = []
    l = 0
    while f"{prefix}/L{l}/rows" in golden:
        layers.append({k: golden[f"{prefix}/L{l}/{k}"]
                       for k in ("rows", "cols", "values", "src_ids", "dst_ids")})
        l += 1
    return (golden[f"{prefix}/targets"], layers, bytes(golden[f"{prefix}/digest"]).hex(),
            golden[f"{prefix}/hits"])


def batch_prefixes(golden):
    out = []
    for k in golden:
        if k.endswith("/digest"):
            out.append(k[:-len("/digest")])
    return sorted(out)


@pytest.fixture(scope="session")
def golden_epoch():
    return load_golden("epoch.npz")


def epoch_graph(golden, name):
    """G2 / g8 of epoch.npz as a HostGraph with its split masks."""
    g = HostGraph(golden[f"{name}/row_offsets"], golden[f"{name}/col_indices"],
                  golden[f"{name}/features"], golden[f"{name}/labels"],
                  int(golden[f"{name}/labels"].max()) + 1, golden[f"{name}/train_mask"])
    g.val_mask = np.asarray(golden[f"{name}/val_mask"], bool)
    g.test_mask = np.asarray(golden[f"{name}/test_mask"], bool)
    return g


def eval_cases(golden):
    return sorted({k.split("/")[1] for k in golden if k.startswith("eval/")})


def refresh_cases(golden):
    return sorted({k.split("/")[2] for k in golden if k.startswith("refresh/case/")})
