"""GPU: the dense SAGE transforms on both backends (tcgen05 3xTF32 and fp32
FFMA split-K) against an fp64 reference of the same contraction.

mq_sage_transform:     y = h[:, :d_in] [W_top | W_bot]           (nn.py:126-131, re-associated)
mq_sage_transform_bwd: dW = [h^T g_top ; h^T g_bot], dh = g [W_top | W_bot]^T   (nn.py:168-174)
Bar: max|a-b| <= 1e-5 * max|b| (fp32-level; one TF32 pass would miss it).
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2601_04707_b200._lib import lib, ptr  # noqa: E402

RTOL = 1e-5
SHAPES = [  # (rows, d_in, d_out)
    (3262, 602, 64),   # Reddit-shaped layer 0
    (1, 602, 64),
    (129, 100, 64),    # products-shaped layer 0
    (1000, 64, 64),
    (257, 30, 13),     # odd widths: N = 26 padded to 32 on the tensor core
    (0, 64, 64),       # empty frontier
    (1131, 32, 32),    # 3-layer g2 middle layer (36 k blocks -> 18 splits of 2)
    (1323, 16, 32),
    (1118, 32, 32),
    (5000, 64, 64),    # several items per CTA on the forward
    (700, 16, 8),      # N = 16: the narrowest UMMA tile (one 32-column TMEM load)
    (40000, 100, 64),  # many items per CTA: the async ring crosses item boundaries
    (97000, 64, 64),   # products-shaped hidden layer: resident weights (kFwdR)
    (50000, 30, 13),   # resident weights with odd widths (N = 26 padded to 32)
]


def _normwise(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    if b.size == 0:
        return 0.0
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-30)


@pytest.fixture(params=[(1, 2), (1, 3), (1, 1), (0, 2)],
                ids=["tcgen05-tma", "tcgen05-tma-all", "tcgen05-cpasync", "ffma"])
def backend(request):
    old, old_k = lib().mq_get_gemm_backend(), lib().mq_get_tc_kernel()
    lib().mq_set_gemm_backend(request.param[0])
    lib().mq_set_tc_kernel(request.param[1])
    yield request.param[0]
    lib().mq_set_gemm_backend(old)
    lib().mq_set_tc_kernel(old_k)


@pytest.mark.parametrize("rows,d_in,d_out", SHAPES)
def test_transform_fwd_bwd(backend, rows, d_in, d_out):
    rng = np.random.default_rng(rows + d_in + d_out)
    ld = (d_in + 3) // 4 * 4
    m_max = max(rows, 1) + 37  # bound larger than the live count
    h = np.zeros((m_max, ld), np.float32)
    h[:rows, :d_in] = rng.standard_normal((rows, d_in))
    h[:rows, d_in:] = 7.0  # pad columns must not leak into the result
    W = (rng.standard_normal((2 * d_in, d_out)) / np.sqrt(d_in)).astype(np.float32)
    g = np.zeros((m_max, 2 * d_out), np.float32)
    g[:rows] = rng.standard_normal((rows, 2 * d_out))
    dev = "cuda"
    th, tW, tg = (torch.from_numpy(x).to(dev) for x in (h, W, g))
    ty = torch.zeros((m_max, 2 * d_out), dtype=torch.float32, device=dev)
    tdW = torch.zeros_like(tW)
    tdh = torch.zeros((m_max, ld), dtype=torch.float32, device=dev)
    m_dev = torch.tensor([rows], dtype=torch.int32, device=dev)
    scr = torch.zeros(int(lib().mq_sage_fused_scratch_bytes(m_max, d_in, d_out)) // 4 + 1,
                      dtype=torch.float32, device=dev)
    s = torch.cuda.current_stream().cuda_stream
    lib().mq_sage_transform(ptr(th), ld, ptr(m_dev), m_max, d_in, ptr(tW), d_out, ptr(ty),
                            ptr(scr), None, None, s)
    y = ty.cpu().numpy()[:rows]
    lib().mq_sage_transform_bwd(ptr(th), ld, ptr(m_dev), m_max, d_in, ptr(tW), d_out, ptr(tg),
                                ptr(tdW), ptr(tdh), ld, ptr(scr), None, None, s)
    torch.cuda.synchronize()
    h64 = h[:rows, :d_in].astype(np.float64)
    W64 = W.astype(np.float64)
    Wcat = np.concatenate([W64[:d_in], W64[d_in:]], axis=1)  # [W_top | W_bot]
    ref_y = h64 @ Wcat
    assert _normwise(y, ref_y) <= RTOL
    g64 = g[:rows].astype(np.float64)
    ref_dW = np.concatenate([h64.T @ g64[:, :d_out], h64.T @ g64[:, d_out:]], axis=0)
    assert _normwise(tdW.cpu().numpy(), ref_dW) <= RTOL
    ref_dh = g64 @ Wcat.T
    assert _normwise(tdh.cpu().numpy()[:rows, :d_in], ref_dh) <= RTOL


def test_tf32_single_pass_would_fail():
    """Sanity of the bar: rounding the operands to TF32 once breaks 1e-5."""
    rng = np.random.default_rng(0)
    h = rng.standard_normal((512, 602)).astype(np.float32)
    W = rng.standard_normal((602, 128)).astype(np.float32)

    def tf32(x):
        u = x.view(np.uint32).astype(np.uint64)
        u = ((u + 0x1000) & 0xFFFFE000).astype(np.uint32)
        return u.view(np.float32)

    exact = h.astype(np.float64) @ W.astype(np.float64)
    one_pass = tf32(h).astype(np.float64) @ tf32(W).astype(np.float64)
    assert _normwise(one_pass, exact) > RTOL


@pytest.fixture(params=[2, 3, 1], ids=["tma", "tma-all", "cpasync"])
def tc_kernel(request):
    old = lib().mq_get_tc_kernel()
    lib().mq_set_tc_kernel(request.param)
    yield request.param
    lib().mq_set_tc_kernel(old)


@pytest.mark.parametrize("rows,d_in,d_out", [(1131, 32, 32), (3262, 602, 64)])
def test_transform_bwd_deterministic(tc_kernel, rows, d_in, d_out):
    """Two runs of the tcgen05 weight gradient give bit-identical results."""
    rng = np.random.default_rng(5)
    ld = (d_in + 3) // 4 * 4
    h = torch.from_numpy(rng.standard_normal((rows, ld)).astype(np.float32)).cuda()
    W = torch.from_numpy(rng.standard_normal((2 * d_in, d_out)).astype(np.float32)).cuda()
    g = torch.from_numpy(rng.standard_normal((rows, 2 * d_out)).astype(np.float32)).cuda()
    m_dev = torch.tensor([rows], dtype=torch.int32, device="cuda")
    scr = torch.zeros(int(lib().mq_sage_fused_scratch_bytes(rows, d_in, d_out)) // 4 + 1,
                      dtype=torch.float32, device="cuda")
    outs = []
    for _ in range(3):
        dW = torch.zeros_like(W)
        lib().mq_sage_transform_bwd(ptr(h), ld, ptr(m_dev), rows, d_in, ptr(W), d_out, ptr(g),
                                    ptr(dW), None, ld, ptr(scr), None, None,
                                    torch.cuda.current_stream().cuda_stream)
        outs.append(dW.cpu())
    assert torch.equal(outs[0], outs[1]) and torch.equal(outs[0], outs[2])


@pytest.mark.parametrize("rows,d_in,d_out", [(2604, 100, 64), (777, 16, 16), (97, 64, 8),
                                             (30000, 100, 64), (0, 16, 16),
                                             (100000, 100, 64), (60000, 16, 16)])
def test_aggregate_first_layer(tc_kernel, rows, d_in, d_out):
    """mq_sage_linear_af (act = relu([agg | h] W)) and mq_sage_linear_af_bwd
    (dW = [agg | h]^T (dh * (act > 0))) against fp64."""
    rng = np.random.default_rng(rows + d_in)
    dev = "cuda"
    agg = rng.standard_normal((max(rows, 1), d_in)).astype(np.float32)
    h = rng.standard_normal((max(rows, 1), d_in)).astype(np.float32)
    W = (rng.standard_normal((2 * d_in, d_out)) / np.sqrt(d_in)).astype(np.float32)
    dh = rng.standard_normal((max(rows, 1), d_out)).astype(np.float32)
    t = lambda a: torch.as_tensor(a, device=dev)
    ag, hh, Wt, dht = t(agg), t(h), t(W), t(dh)
    act = torch.zeros((max(rows, 1), d_out), device=dev)
    m = torch.tensor([rows], dtype=torch.int32, device=dev)
    part = torch.zeros(int(lib().mq_sage_af_parts_bytes(max(rows, 1), d_out)) // 4 + 1, device=dev)
    s = torch.cuda.current_stream().cuda_stream
    lib().mq_sage_linear_af(ptr(ag), d_in, ptr(hh), d_in, ptr(m), max(rows, 1), d_in, ptr(Wt),
                            d_out, ptr(act), d_out, ptr(part), s)
    z = np.concatenate([agg, h], 1).astype(np.float64)[:rows] @ W.astype(np.float64)
    ref_act = np.maximum(z, 0)
    got = act.cpu().numpy()[:rows]
    assert _normwise(got, ref_act) <= RTOL
    dwp = torch.zeros(int(lib().mq_sage_af_dw_parts_bytes(d_in, d_out)) // 4 + 1, device=dev)
    nparts = torch.zeros(1, dtype=torch.int32, device=dev)
    lib().mq_sage_linear_af_bwd(ptr(ag), d_in, ptr(hh), d_in, ptr(m), max(rows, 1), d_in, ptr(dht),
                                d_out, ptr(act), d_out, d_out, ptr(dwp), ptr(nparts), s)
    S = int(nparts.item())
    dw = dwp[:S * 2 * d_in * d_out].view(S, 2 * d_in, d_out).sum(0).cpu().numpy()
    dz = dh[:rows].astype(np.float64) * (got > 0)
    ref_dw = np.concatenate([agg, h], 1).astype(np.float64)[:rows].T @ dz
    assert _normwise(dw, ref_dw) <= 2 * RTOL


@pytest.mark.parametrize("rows,d_in,d_out", [(3262, 602, 64), (1131, 32, 32), (1000, 64, 64),
                                             (1323, 16, 32), (97, 64, 8)])
def test_deferred_partials_repeated(rows, d_in, d_out):
    """The deferred transform / weight-gradient partials (the fused step's
    path; bulk async-copy epilogue on each CTA's last tile), summed over the
    published split count, against fp64 -- 20 repetitions, since a staging
    buffer reused while its previous copy still reads it shows up only
    intermittently."""
    rng = np.random.default_rng(rows * 7 + d_in)
    ld = (d_in + 3) // 4 * 4
    h = np.zeros((rows, ld), np.float32)
    h[:, :d_in] = rng.standard_normal((rows, d_in))
    W = (rng.standard_normal((2 * d_in, d_out)) / np.sqrt(d_in)).astype(np.float32)
    g = rng.standard_normal((rows, 2 * d_out)).astype(np.float32)
    th, tW, tg = (torch.from_numpy(x).cuda() for x in (h, W, g))
    m_dev = torch.tensor([rows], dtype=torch.int32, device="cuda")
    scr = torch.zeros(int(lib().mq_sage_fused_scratch_bytes(rows, d_in, d_out)) // 4 + 1,
                      dtype=torch.float32, device="cuda")
    yp = torch.zeros(int(lib().mq_sage_y_parts_bytes(rows, d_out)) // 4 + 1, dtype=torch.float32,
                     device="cuda")
    dwp = torch.zeros(int(lib().mq_sage_dw_parts_bytes(d_in, d_out)) // 4 + 1,
                      dtype=torch.float32, device="cuda")
    ny = torch.zeros(1, dtype=torch.int32, device="cuda")
    nw = torch.zeros(1, dtype=torch.int32, device="cuda")
    h64, W64, g64 = h[:, :d_in].astype(np.float64), W.astype(np.float64), g.astype(np.float64)
    ref_y = h64 @ np.concatenate([W64[:d_in], W64[d_in:]], axis=1)
    ref_dw = np.concatenate([h64.T @ g64[:, :d_out], h64.T @ g64[:, d_out:]], axis=0)
    s = torch.cuda.current_stream().cuda_stream
    for _ in range(20):
        lib().mq_sage_transform(ptr(th), ld, ptr(m_dev), rows, d_in, ptr(tW), d_out, None,
                                ptr(scr), ptr(yp), ptr(ny), s)
        lib().mq_sage_transform_bwd(ptr(th), ld, ptr(m_dev), rows, d_in, ptr(tW), d_out, ptr(tg),
                                    None, None, ld, ptr(scr), ptr(dwp), ptr(nw), s)
        torch.cuda.synchronize()
        S = int(ny.item())
        y = yp[:S * rows * 2 * d_out].view(S, rows, 2 * d_out).double().sum(0).cpu().numpy()
        assert _normwise(y, ref_y) <= RTOL
        S = int(nw.item())
        p = dwp[:S * d_in * 2 * d_out].view(S, d_in, 2 * d_out).double().sum(0).cpu().numpy()
        dw = np.concatenate([p[:, :d_out], p[:, d_out:]], axis=0)
        assert _normwise(dw, ref_dw) <= RTOL
