"""Pin the layer-wise oracle (LADIES / FastGCN, flat / debias / replace, and
the GCN node-wise arm) to vectors the reference itself produced
(``tests/golden/make_golden_layerwise.py``).  CPU only."""

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import layerwise as olw
from oracle import sampler as osamp

LW = np.load(GOLDEN / "layerwise.npz")


def _graph(name):
    ro = LW[f"graph/{name}/row_offsets"]
    ci = LW[f"graph/{name}/col_indices"]
    return ro, ci, LW[f"graph/{name}/a_hat_degrees"]


def _run_case(case):
    ro, ci, dh = _graph(str(LW[f"{case}/graph"]))
    budget, layers, flat, debias, replace = LW[f"{case}/params"].tolist()
    seed, epoch, batch = LW[f"{case}/key"].tolist()
    rng = olw.LayerRng(seed, epoch, batch)
    method = str(LW[f"{case}/method"])
    targets = np.asarray(LW[f"{case}/target_ids"])
    dropped = 0
    if method == "ladies":
        # the fixture stores the kept targets; rebuild the request with the
        # dropped ones for the g9 case (an isolated node 8 asked twice)
        req = np.array([8, 1, 8, 6]) if case == "g9_ladies_drop" else targets
        blocks, dropped = olw.sample_ladies(ro, ci, req, budget, layers, rng, flat=bool(flat),
                                            debias=bool(debias), replace=bool(replace),
                                            deg_hat=dh)
    else:
        blocks = olw.sample_fastgcn(ro, ci, targets, budget, layers, rng, flat=bool(flat),
                                    debias=bool(debias), deg_hat=dh)
    assert rng.calls == layers
    return blocks, dropped


@pytest.mark.parametrize("case", [str(c) for c in LW["cases"]])
def test_layerwise_blocks_match_reference(case):
    blocks, dropped = _run_case(case)
    assert dropped == int(LW[f"{case}/dropped"])
    for l, blk in enumerate(blocks):
        for k in ("rows", "cols", "values", "effective_values", "src_ids", "dst_ids"):
            ref = LW[f"{case}/L{l}/{k}"]
            got = getattr(blk, k)
            assert got.dtype.kind == ref.dtype.kind, (k, got.dtype, ref.dtype)
            np.testing.assert_array_equal(got, ref, err_msg=f"{case} L{l} {k}")
        np.testing.assert_array_equal(blk.sample_probs, LW[f"{case}/L{l}/sample_probs"])
    kept = blocks[-1].dst_ids
    d = osamp.digest_of(kept, blocks, LW[f"{case}/features"])
    assert bytes.fromhex(d) == LW[f"{case}/digest"].tobytes()


@pytest.mark.parametrize("g", ["g8", "g2"])
def test_probabilities_match_reference(g):
    ro, ci, dh = _graph(g)
    prev, cand = LW[f"probs/{g}/prev"], LW[f"probs/{g}/cand"]
    np.testing.assert_array_equal(olw.candidates_of(ro, ci, prev), cand)
    np.testing.assert_array_equal(olw.layer_probs(ro, ci, dh, cand, prev, flat=False),
                                  LW[f"probs/{g}/ladies"])
    np.testing.assert_array_equal(olw.layer_probs(ro, ci, dh, cand, prev, flat=True),
                                  LW[f"probs/{g}/flat"])
    np.testing.assert_array_equal(olw.fastgcn_probs(ro, ci, dh), LW[f"probs/{g}/fastgcn"])
    np.testing.assert_array_equal(olw.fastgcn_probs(ro, ci, dh, flat=True),
                                  LW[f"probs/{g}/fastgcn_flat"])
    np.testing.assert_array_equal(olw.a_hat_degrees(ro, ci), dh)


def test_debias_coefficients_match_reference():
    got = olw.debias_coefficients(LW["debias/probs"], int(LW["debias/n"]))
    np.testing.assert_array_equal(got, LW["debias/coef"])


@pytest.mark.parametrize("case", [str(c) for c in LW["gcn_cases"]])
def test_gcn_node_wise_arm_matches_reference(case):
    g = case.split("_")[1]
    ro, ci, dh = _graph(g)
    seed, epoch, batch = 5, 2, 9
    fo = LW[f"{case}/fanouts"].tolist()
    sage = osamp.sample_node_wise(ro, ci, LW[f"{case}/target_ids"], fo, seed=seed, epoch=epoch,
                                  batch_id=batch)
    for l, blk in enumerate(sage):
        rows, cols, vals = olw.gcn_block_values(ro, ci, dh, blk)
        np.testing.assert_array_equal(rows, LW[f"{case}/L{l}/rows"])
        np.testing.assert_array_equal(cols, LW[f"{case}/L{l}/cols"])
        np.testing.assert_array_equal(vals, LW[f"{case}/L{l}/values"])
        np.testing.assert_array_equal(blk.src_ids, LW[f"{case}/L{l}/src_ids"])


def test_layer_rng_contract():
    """random(n) is a prefix-stable stream per layer; choice follows NumPy's
    cdf / searchsorted algorithm over the same uniforms."""
    r = olw.LayerRng(1, 2, 3)
    u = r.random(10)
    assert r.calls == 1 and ((u >= 0) & (u < 1)).all()
    np.testing.assert_array_equal(olw.layer_uniforms(1, 2, 3, 0, 4), u[:4])
    p = np.array([0.1, 0.0, 0.6, 0.3])
    idx = r.choice(4, size=50, replace=True, p=p)
    cdf = np.cumsum(p)
    cdf /= cdf[-1]
    np.testing.assert_array_equal(idx, np.searchsorted(cdf, olw.layer_uniforms(1, 2, 3, 1, 50),
                                                       side="right"))
    assert not np.any(idx == 1)
