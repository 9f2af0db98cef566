"""Micro-benchmark of the tcgen05 GEMM entry points on synthetic operands
(GPU): FWD (mq_full_transform, Y = h [W_top|W_bot]) and the aggregate-first
FCAT / DCAT modes, CUDA-event timed.  With the MQ_TC_TRACE library
(MQGNN_LIB=.../libmqgnn_trace.so) also prints CTA 0's phase timeline."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from paper_2601_04707_b200._lib import lib, ptr  # noqa: E402


def timeit(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) * 1e3 / reps


def trace():
    if not hasattr(lib().dll, "mq_debug_tc_trace"):
        return ""
    if lib().mq_get_tc_kernel() >= 2:
        buf = (C.c_ulonglong * 64)()
        lib().dll.mq_debug_tc_trace(buf)
        t = [int(x) for x in buf]
        rel = lambda i: (t[i] - t[0]) / 1e3 if t[i] >= t[0] and t[i] - t[0] < 1e9 else float("nan")
        f = lambda a, b: " ".join(f"{rel(i):6.2f}" for i in range(a, b))
        return (f"\n      setup {rel(1):.2f}  end {rel(29):.2f}\n      tma  {f(2, 10)}\n      conv {f(10, 18)}"
                f"  done0/1 {rel(30):.2f} {rel(31):.2f}\n      mma  {f(18, 26)}\n      epi  acc0 {rel(26):.2f}"
                f" st0 {rel(27):.2f} acc1 {rel(28):.2f}\n      conv1 phases (full, A split, tmem st, B ld, bar, B st, fence) "
                f"{rel(11):.2f} {f(32, 38)}")
    buf = (C.c_ulonglong * 64)()
    lib().dll.mq_debug_tc_trace(buf)
    t = [int(x) for x in buf]
    base = t[0]
    rel = lambda i: (t[i] - base) / 1e3 if t[i] >= base and t[i] - base < 1e9 else float("nan")
    out = f"\n      setup {rel(1):.2f} item0 {rel(2):.2f}"
    for it in range(3):
        out += f"\n      kb{it}: " + " ".join(f"{rel(3 + 8 * it + p):.2f}" for p in range(8))
    out += f"\n      acc {rel(27):.2f} epi {rel(28):.2f} end {rel(29):.2f}"
    cta = (C.c_ulonglong * 512)()
    lib().dll.mq_debug_tc_cta(cta)
    st = [int(cta[2 * i]) for i in range(148)]
    en = [int(cta[2 * i + 1]) for i in range(148)]
    t0 = min(st)
    starts = sorted((x - t0) / 1e3 for x in st)
    ends = sorted((x - t0) / 1e3 for x in en)
    out += (f"\n      CTA start min/med/max {starts[0]:.1f}/{starts[74]:.1f}/{starts[-1]:.1f} us,"
            f" end min/med/max {ends[0]:.1f}/{ends[74]:.1f}/{ends[-1]:.1f} us")
    return out


dev = "cuda"
s = torch.cuda.current_stream().cuda_stream
VERSIONS = [int(v) for v in os.environ.get("MQ_TC_VERSIONS", "1,3").split(",")]


def bwd(M, K, N):
    """mq_sage_transform_bwd: dW (DW mode, K = rows) + dh (DX mode)."""
    ld = (K + 3) // 4 * 4
    h = torch.randn(M, ld, device=dev)
    W = torch.randn(2 * K, N, device=dev)
    g = torch.randn(M, 2 * N, device=dev)
    dW = torch.empty_like(W)
    dh = torch.empty(M, ld, device=dev)
    m_dev = torch.tensor([M], dtype=torch.int32, device=dev)
    scr = torch.empty(int(lib().mq_sage_fused_scratch_bytes(M, K, N)) // 4 + 1, device=dev)
    us = timeit(lambda: lib().mq_sage_transform_bwd(ptr(h), ld, ptr(m_dev), M, K, ptr(W), N, ptr(g),
                                                    ptr(dW), ptr(dh), ld, ptr(scr), None, None, s))
    byt = 4 * (M * ld + M * 2 * N + M * ld)
    print(f"BWD  M={M:7d} K={K:4d} N={2*N:4d}: {us:8.1f} us  {byt / us / 1e3:7.1f} GB/s (dW + dh)")
    us = timeit(lambda: lib().mq_sage_transform_bwd(ptr(h), ld, ptr(m_dev), M, K, ptr(W), N, ptr(g),
                                                    ptr(dW), None, ld, ptr(scr), None, None, s))
    byt = 4 * (M * ld + M * 2 * N)
    print(f"DW   M={K:7d} K={M:6d} N={2*N:4d}: {us:8.1f} us  {byt / us / 1e3:7.1f} GB/s  {trace()}")


for ver in VERSIONS:
  lib().mq_set_tc_kernel(ver)
  print(f"--- tc kernel v{ver}")
  for (M, K, N) in [(2604, 602, 64), (97297, 64, 64), (12700, 64, 64)]:
    bwd(M, K, N)
  for (M, K, N) in [(2604, 602, 64), (97297, 100, 64), (337394, 100, 64), (97297, 64, 64)]:
      ld = (K + 3) // 4 * 4
      h = torch.randn(M, ld, device=dev)
      W = torch.randn(2 * K, N, device=dev)
      y = torch.empty(M, 2 * N, device=dev)
      part = torch.empty(int(lib().mq_full_transform_part_floats(M, N)), device=dev)
      us = timeit(lambda: lib().mq_full_transform(ptr(h), ld, M, K, ptr(W), N, ptr(y), ptr(part), s))
      byt = 4 * (M * ld + 2 * K * N + 2 * M * 2 * N)  # incl. the S=1 reduce copy
      print(f"FWD  M={M:7d} K={K:4d} N={2*N:4d}: {us:8.1f} us  {byt / us / 1e3:7.1f} GB/s  {trace()}")
      # aggregate-first forward: [agg | h] (M x 2K) W (2K x N)
      m_dev = torch.tensor([M], dtype=torch.int32, device=dev)
      agg = torch.randn(M, ld, device=dev)
      act = torch.empty(M, N, device=dev)
      W2 = torch.randn(2 * ld, N, device=dev)
      if K % 4 == 0:
          pa = torch.empty(int(lib().mq_sage_af_parts_bytes(M, N)) // 4 + 1, device=dev)
          us = timeit(lambda: lib().mq_sage_linear_af(ptr(agg), ld, ptr(h), ld, ptr(m_dev), M, K,
                                                      ptr(W2), N, ptr(act), N, ptr(pa), s))
          byt = 4 * (2 * M * ld + 2 * M * N)
          print(f"FCAT M={M:7d} K={2*K:4d} N={N:4d}: {us:8.1f} us  {byt / us / 1e3:7.1f} GB/s  {trace()}")
          dh = torch.randn(M, N, device=dev)
          npd = torch.zeros(1, dtype=torch.int32, device=dev)
          pd = torch.empty(int(lib().mq_sage_af_dw_parts_bytes(K, N)) // 4 + 1, device=dev)
          us = timeit(lambda: lib().mq_sage_linear_af_bwd(ptr(agg), ld, ptr(h), ld, ptr(m_dev), M, K,
                                                          ptr(dh), N, ptr(act), N, N, ptr(pd),
                                                          ptr(npd), s))
          byt = 4 * (2 * M * ld + 2 * M * N)
          print(f"DCAT M={2*K:7d} K={M:6d} N={N:4d}: {us:8.1f} us  {byt / us / 1e3:7.1f} GB/s  "
                f"S={int(npd.item())} {trace()}")
