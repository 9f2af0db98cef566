"""CPU: the algorithmic byte / flop models behind bench.py's roofline
(profiling.op_models) on a products-shaped
3-layer count set: every train op of both input-layer associations has a
model, the numbers are the closed forms, and no model exceeds the bytes the
op can touch (a bytes-for-flops slip once made a roofline read 6x the HBM
peak)."""

from paper_2601_04707_b200.profiling import op_models

COUNTS = {"n_targets": 1024,
          "hops": [[1024, 12700, 14662], [12700, 97297, 126851], [97297, 337394, 486476]]}
DIMS = [100, 64, 64, 47]


def _models():
    return op_models(COUNTS, DIMS, (15, 10, 5), 8, True, 27008, 47, 100)


def test_every_fused_op_has_a_model():
    m = _models()
    for name in ("sage_transform_l0", "sage_aggregate_l0", "sage_scatter_bwd_l0",
                 "sage_transform_bwd_l0", "sage_transform_l1", "sage_transform_bwd_l1",
                 "sage_spmm_l0", "sage_linear_af_l0", "sage_linear_af_bwd_l0", "sage_head",
                 "optimizer", "prep_sample", "prep_relabel", "prep_gather"):
        assert name in m and m[name]["bytes"] > 0, name


def test_closed_forms():
    m = _models()
    nd, ns, nnz = COUNTS["hops"][2]
    d, dout = DIMS[0], DIMS[1]
    assert m["sage_linear_af_l0"]["bytes"] == 4 * (nd * 2 * d + 2 * d * dout + nd * dout)
    assert m["sage_linear_af_l0"]["flops"] == 2.0 * nd * 2 * d * dout
    assert m["sage_spmm_l0"]["bytes"] == 4 * d * (nnz + nd) + 8 * nnz + 4 * (nd + 1)
    nd1, ns1, _ = COUNTS["hops"][1]
    d1, do1 = DIMS[1], DIMS[2]
    # layer 1 backward: dW = h^T G plus dh = G W^T (one more read of G and W, one write of dh)
    assert m["sage_transform_bwd_l1"]["bytes"] == (4 * (ns1 * d1 + ns1 * 2 * do1 + 2 * d1 * do1)
                                                  + 4 * (ns1 * 2 * do1 + 2 * d1 * do1 + ns1 * d1))
    assert m["sage_transform_bwd_l1"]["flops"] == 2 * (2.0 * ns1 * d1 * 2 * do1)


def test_models_stay_within_touchable_bytes():
    """No op's algorithmic bytes exceed (everything one batch can read or
    write) x 3, times the Q = 8 batches a prep launch covers."""
    m = _models()
    big = 4 * (337394 * 100 * 2 + 97297 * 64 * 8 + 486476 * 16)
    for name, v in m.items():
        q = 8 if name.startswith("prep_") else 1
        assert v["bytes"] <= 3 * big * q, (name, v["bytes"])


def test_sector_models_of_the_random_access_prep():
    """prep_sample / prep_relabel also carry a 32-byte-sector count (one
    sector per random touch on top of the compulsory bytes)."""
    m = _models()
    hops, Q, L = COUNTS["hops"], 8, 3
    relab_sec = sum(32 * (3 * nnz + (ns - nd) + (nd if h == 0 else 0) + (ns if h == L - 1 else 0))
                    for h, (nd, ns, nnz) in enumerate(hops))
    assert m["prep_relabel"]["sector_bytes"] == m["prep_relabel"]["bytes"] + Q * relab_sec
    samp_sec = sum(32 * (2 * nd + 2 * nnz) for nd, ns, nnz in hops)  # cached: hot offsets / arcs
    assert m["prep_sample"]["sector_bytes"] == m["prep_sample"]["bytes"] + Q * samp_sec
    for k in ("prep_sample", "prep_relabel"):
        assert m[k]["sector_bytes"] > m[k]["bytes"]
