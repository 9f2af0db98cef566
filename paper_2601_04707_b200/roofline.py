"""Algorithmic byte / flop models of the step's kernels.

Each model returns the compulsory DRAM traffic (bytes) of ONE launch given
the step's device counts, following SURVEY.md §8(d) where the algorithm is
the same and stating the B200 variant where it differs (the sampler reads
O(fanout) entries per row through the residency index instead of scanning
whole rows).  Used by ``bench.py`` to turn CUDA-event kernel times into
achieved GB/s against the measured HBM peak.
"""

from __future__ import annotations


def step_models(counts: dict, dims: list, fanouts: tuple, cached: bool, n_params: int,
                num_classes: int) -> dict:
    """{kernel name: [bytes per launch, ...] in launch order} for one step.

    counts: {"n_targets": B, "hops": [(n_dst, n_src, nnz), ...]} (hop 0 = seeds)
    dims:   [d_in, hidden..., classes]
    """
    L = len(fanouts)
    hops = counts["hops"]
    B = counts["n_targets"]
    m: dict = {}

    def add(name, b):
        m.setdefault(name, []).append(float(b))

    add("batch_setup", 8 * B)
    for h, (nd, ns, nnz) in enumerate(hops):
        # K1: dst id + row offsets (+ hot offsets) per row, output ids + count;
        # per pick one column read (+ one hot-arc index when cached)
        add("sample_hop", nd * (4 + 16 + (16 if cached else 0) + 4) + nnz * (4 + 4 + (8 if cached else 0)))
        # K2 (§8d): i*(nnz + n_dst) read + i*(nnz + n_src) + 4*(n_dst+1) written
        add("relabel_mark", 4 * nd * 3)
        add("relabel_first", 4 * nnz * 3)
        add("relabel_flag_scan", 4 * nnz * 3 + 4 * (ns - nd) * 2)
        add("relabel_cols", 4 * nnz * 5)
        add("relabel_clean", 4 * ns * 3)
        add("scan", 4 * nd + 4 * (nd + 1))
    nd_in, ns_in, _ = hops[-1]
    d0 = dims[0]
    # K3: d-float row read + write per input row, id + slot lookup
    add("gather", 2 * 4 * d0 * ns_in + 8 * ns_in)
    for l in range(L):
        nd, ns, nnz = hops[L - 1 - l]
        d, dout = dims[l], dims[l + 1]
        # K4 compulsory: every src row read once, every dst row written once,
        # triplets and row pointers read
        add("spmm_fwd", 4 * d * (ns + nd) + 8 * nnz + 4 * (nd + 1))
        add("linear_fwd", 4 * (nd * 2 * d + 2 * d * dout + nd * dout * (2 if l < L - 1 else 1)))
    add("gather_labels", 12 * B)
    add("softmax_ce", 4 * B * num_classes * 2 + 4 * B)
    for l in range(L - 1, -1, -1):
        nd, ns, nnz = hops[L - 1 - l]
        d, dout = dims[l], dims[l + 1]
        add("linear_bwd_w", 4 * (nd * 2 * d + nd * dout))
        add("linear_bwd_w_reduce", 4 * 2 * d * dout)
        if l > 0:
            add("linear_bwd_x", 4 * (nd * dout + 2 * d * dout + nd * 2 * d))
            add("spmm_bwd_init", 4 * d * (nd + ns))
            add("spmm_bwd_scatter", 4 * d * (nd + ns) + 12 * nnz)
            add("spmm_bwd_mask", 4 * d * ns * 3)
    add("adam", 4 * n_params * 7)
    add("step_bump", 4)
    return m


def step_flops(counts: dict, dims: list, fanouts: tuple) -> dict:
    """GEMM flops (2*M*K*N) of the dense transforms of one step."""
    L = len(fanouts)
    hops = counts["hops"]
    out = {"linear_fwd": 0.0, "linear_bwd_w": 0.0, "linear_bwd_x": 0.0}
    for l in range(L):
        nd = hops[L - 1 - l][0]
        k, n = 2 * dims[l], dims[l + 1]
        out["linear_fwd"] += 2.0 * nd * k * n
        out["linear_bwd_w"] += 2.0 * nd * k * n
        if l > 0:
            out["linear_bwd_x"] += 2.0 * nd * k * n
    return out
