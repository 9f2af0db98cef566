"""ctypes binding of libmqgnn.so (the C-ABI in include/mqgnn.h).

The product path has no CPU fallback: if the library is missing or a call
fails, an ``MQError`` is raised.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "libmqgnn.so"

P = C.c_void_p
I32 = C.c_int32
I64 = C.c_int64
U32 = C.c_uint32
U64 = C.c_uint64
F32 = C.c_float
F64 = C.c_double

MQ_GRAD_MAX_SEG = 8


class GradSeg(C.Structure):
    """mq_grad_seg (include/mqgnn.h): one deferred split-K gradient range."""
    _fields_ = [("part", P), ("nparts_dev", P), ("stride", I64), ("offset", I64), ("size", I64),
                ("nparts", I32), ("kind", I32), ("d_in", I32), ("d_out", I32)]


class GradSrc(C.Structure):
    """mq_grad_src: up to MQ_GRAD_MAX_SEG segments resolved by the optimizer kernels."""
    _fields_ = [("nseg", I32), ("pad_", I32), ("seg", GradSeg * MQ_GRAD_MAX_SEG)]


# name -> (restype, argtypes); mirrors include/mqgnn.h one to one
SIGNATURES = {
    "mq_version": (C.c_int, []),
    "mq_last_error": (C.c_char_p, []),
    "mq_stream_check": (C.c_int, [P]),
    "mq_philox_fill_host": (C.c_int, [U64, U64, U32, U32, U32, U32, P]),
    "mq_philox_fill": (C.c_int, [U64, U64, U32, U32, U32, U32, P, P]),
    "mq_fisher_yates_host": (C.c_int, [U64, U64, U32, U32, U32, I64, I32, P]),
    "mq_scan_scratch_bytes": (I64, [I64]),
    "mq_strip_self_loops": (C.c_int, [P, P, I64, I64, P, P, P, P]),
    "mq_residency_index": (C.c_int, [P, P, I64, I64, P, P, P, P, P, P]),
    "mq_residency_slots": (C.c_int, [P, I64, P, P, P, P]),
    "mq_sample_hop": (C.c_int, [P, P, P, P, P, P, I32, I32, U64, U64, U32, U32, P, P, P, P]),
    "mq_batch_setup": (C.c_int, [P, I64, I32, I32, I32, P, P, P, P, P]),
    "mq_step_commit": (C.c_int, [P, P, I32, P, I32, P]),
    "mq_relabel_scratch_bytes": (I64, [I32, I32]),
    "mq_relabel": (C.c_int, [P, P, I32, P, P, I32, P, P, P, P, P, P, P, P, P, P]),
    "mq_gather": (C.c_int, [P, I32, P, P, I32, P, P, I32, I32, P, I32, P, P]),
    "mq_spmm_fwd": (C.c_int, [P, P, P, P, I32, P, I32, I32, P, I32, P]),
    "mq_spmm_bwd": (C.c_int, [P, P, P, P, I32, P, I32, P, I32, I32, P, I32, P, I32, P]),
    "mq_sage_linear_fwd": (C.c_int, [P, I32, P, I32, P, I32, I32, P, I32, P, I32, P, I32, P, P]),
    "mq_linear_scratch_bytes": (I64, [I32, I32, I32]),
    "mq_sage_linear_bwd": (C.c_int, [P, I32, P, I32, P, I32, I32, P, I32, P, I32, P, P, I32,
                                     P, P]),
    "mq_softmax_ce": (C.c_int, [P, I32, P, P, I32, I32, P, I32, P, P, P]),
    "mq_gather_labels": (C.c_int, [P, P, P, I32, P, P]),
    "mq_adam": (C.c_int, [P, P, P, P, P, F64, I64, P, P, I32, P, P, P, P]),
    "mq_sgd": (C.c_int, [P, P, P, F64, I64, P, P, P, P, P]),
    "mq_f32_to_f64": (C.c_int, [P, P, I64, P]),
    "mq_pack_grads": (C.c_int, [P, I64, P, P, P, P]),
    "mq_grad_reduce": (C.c_int, [P, P, I64, P, P]),
    "mq_f64_to_f32": (C.c_int, [P, F64, P, I64, P]),
    "mq_scan_i32": (C.c_int, [P, P, I32, P, P, P]),
    "mq_sage_fused_scratch_bytes": (I64, [I32, I32, I32]),
    "mq_sage_y_deferred": (C.c_int, [I32]),
    "mq_sage_y_parts_bytes": (I64, [I32, I32]),
    "mq_sage_transform": (C.c_int, [P, I32, P, I32, I32, P, I32, P, P, P, P, P]),
    "mq_sage_aggregate": (C.c_int, [P, P, P, P, I32, P, I32, P, P, P, I32, P, P, I32, P, P, I32,
                                    P]),
    "mq_sage_scatter_bwd": (C.c_int, [P, P, P, P, I32, P, I32, P, I32, I32, P, P]),
    "mq_sage_dw_deferred": (C.c_int, [I32]),
    "mq_sage_dw_parts_bytes": (I64, [I32, I32]),
    "mq_sage_transform_bwd": (C.c_int, [P, I32, P, I32, I32, P, I32, P, P, P, I32, P, P, P, P]),
    "mq_sage_dw_grad_seg": (C.c_int, [P, P, I32, I32, I64, P]),
    "mq_sage_head_grad_seg": (C.c_int, [I32, I32, I32, P, I64, P]),
    "mq_sage_head_scratch_bytes": (I64, [I32, I32, I32]),
    "mq_sage_head": (C.c_int, [P, P, P, P, I32, P, I32, I32, P, I32, P, P, P, I32, P, P, I32, P,
                               I32, P, P, P]),
    "mq_set_gemm_backend": (C.c_int, [I32]),
    "mq_get_gemm_backend": (C.c_int, []),
    "mq_set_pdl": (C.c_int, [I32]),
    "mq_set_tc_grid_cap": (C.c_int, [I32]),
    "mq_set_tc_kernel": (C.c_int, [I32]),
    "mq_get_tc_kernel": (C.c_int, []),
    "mq_memcpy_async": (C.c_int, [P, P, I64, P]),
    "mq_memset_async": (C.c_int, [P, I32, I64, P]),
    "mq_get_pdl": (C.c_int, []),
    "mq_sage_af_parts_bytes": (I64, [I32, I32]),
    "mq_sage_af_dw_parts_bytes": (I64, [I32, I32]),
    "mq_sage_linear_af": (C.c_int, [P, I32, P, I32, P, I32, I32, P, I32, P, I32, P, P]),
    "mq_sage_linear_af_bwd": (C.c_int, [P, I32, P, I32, P, I32, I32, P, I32, P, I32, I32, P, P,
                                        P]),
    "mq_full_transform_part_floats": (I64, [I64, I32]),
    "mq_full_transform": (C.c_int, [P, I32, I64, I32, P, I32, P, P, P]),
    "mq_full_agg_scratch_bytes": (I64, [I64, I32]),
    "mq_full_aggregate": (C.c_int, [P, P, I64, I64, P, I32, I32, I32, P, I32, P, P]),
    "mq_accuracy": (C.c_int, [P, I32, I32, P, P, I64, P, P]),
    "mq_full_transform_half": (C.c_int, [P, I32, I64, I32, P, I32, P, I32, P, P]),
    "mq_full_aggregate_inplace": (C.c_int, [P, P, I64, I64, P, I32, I32, I32, P, I32, P, P]),
    "mq_full_aggregate_rows": (C.c_int, [P, P, I64, I64, P, I32, I32, P, P, I32, P, P]),
    "mq_full_linear_cat_part_floats": (I64, [I64, I32]),
    "mq_full_linear_cat": (C.c_int, [P, I32, P, I32, I64, I32, P, I32, P, I32, I32, P, P]),
    "mq_accuracy_rows": (C.c_int, [P, I32, I32, P, P, I64, P, P]),
    "mq_in_degrees": (C.c_int, [P, I64, I64, P, P, P]),
    "mq_degree_probs": (C.c_int, [P, I64, I64, P, P]),
    "mq_walk_scratch_bytes": (I64, [I64]),
    "mq_walk_probs": (C.c_int, [P, P, I64, P, P, P, I64, I32, I32, P, P, P, P]),
    "mq_refresh_scratch_bytes": (I64, [I64]),
    "mq_refresh_select": (C.c_int, [P, I64, I64, U64, U64, P, P, P, P]),
    "mq_refresh_uniforms_host": (C.c_int, [U64, U64, I64, P]),
    "mq_build_csr_scratch_bytes": (I64, [I64]),
    "mq_build_csr_keys": (C.c_int, [P, I64, I64, P, P, P, P, P]),
    "mq_build_csr_finish": (C.c_int, [P, I64, I64, P, P, P]),
    "mq_narrow_cols": (C.c_int, [P, I64, I64, P, P, P]),
    "mq_degree_buckets": (C.c_int, [P, I64, P, P]),
    "mq_prep_scratch_bytes": (I64, [I32, I32]),
    "mq_prep_batches": (C.c_int, [P, P]),
    "mq_prof_enable": (C.c_int, [C.c_int]),
    "mq_prof_reset": (C.c_int, []),
    "mq_prof_num_kernels": (C.c_int, []),
    "mq_prof_kernel_name": (C.c_char_p, [C.c_int]),
    "mq_prof_read": (C.c_int, [P, P, I32]),
    "mq_launch_count": (I64, []),
    "mq_gather_sharded": (C.c_int, [P, I32, P, P, I32, I32, P, P, I32, I32, P, I32, P, P]),
    "mq_trace_stamp": (C.c_int, [P, I32, P, U32, P, P]),
    "mq_peer_arena_bytes": (I64, [I64, I32]),
    "mq_peer_alloc": (C.c_int, [I64, P]),
    "mq_peer_free": (C.c_int, [P]),
    "mq_ipc_export": (C.c_int, [P, P]),
    "mq_ipc_open": (C.c_int, [P, P]),
    "mq_ipc_close": (C.c_int, [P]),
    "mq_racom_publish": (C.c_int, [P, P, P, P, P]),
    "mq_racom_apply": (C.c_int, [P, I32, I32, P, P, P, P, P, I32, P, P, P]),
    "mq_peer_state": (C.c_int, [P, P, P]),
    "mq_layer_scratch_bytes": (I64, [I64]),
    "mq_layer_entries": (C.c_int, [P, P, P, I32, P, P, P]),
    "mq_layer_live_targets": (C.c_int, [P, P, P, I32, P, P, P, P]),
    "mq_layer_fastgcn_probs": (C.c_int, [P, P, P, I64, I32, P, P, P]),
    "mq_layer_block": (C.c_int, [P, P, P, I64, P, I32, P, I64, P, P, I32, I32, I32, U64, U64,
                                 U32, U32, P, P, P, P, P, P, P, P, P, P, P]),
    "mq_gcn_block": (C.c_int, [P, P, P, P, P, P, I32, P, P, P, P, P]),
    "mq_layer_uniforms_host": (C.c_int, [U64, U64, U32, U32, I64, P]),
    "mq_layer_cdf": (C.c_int, [P, I64, P, P]),
    "mq_relu": (C.c_int, [P, P, I64, P]),
    "mq_sage_linear_dt": (C.c_int, [P, I32, I32, P, I32, P, I32, P, I32, P, P]),
    "mq_gcn_linear_fwd": (C.c_int, [P, I32, P, I32, I32, P, I32, P, I32, P, I32, P, P]),
    "mq_gcn_linear_bwd": (C.c_int, [P, I32, P, I32, I32, P, I32, P, I32, P, P, I32, P, P]),
}

_INT_STATUS = {name for name, (res, _) in SIGNATURES.items()
               if res is C.c_int and name not in ("mq_version", "mq_prof_num_kernels",
                                                       "mq_get_gemm_backend", "mq_get_pdl", "mq_get_tc_kernel",
                                                       "mq_sage_dw_deferred",
                                                       "mq_sage_y_deferred")}


class MQError(RuntimeError):
    """A libmqgnn call failed (argument, CUDA or state error)."""


class MQSamplingError(MQError):
    """MQ_ERR_SAMPLING: the layer-wise sampler's SamplingError (empty
    candidate set, all-zero column norms)."""


MQ_ERR_SAMPLING = 4


class _Lib:
    def __init__(self, path: Path):
        if not path.exists():
            raise MQError(
                f"{path} is missing: build it with `python -m paper_2601_04707_b200._build` "
                "(there is no CPU fallback)")
        self.path = path
        self.dll = C.CDLL(str(path))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(self.dll, name)
            fn.restype = res
            fn.argtypes = args

    def __getattr__(self, name):
        fn = getattr(self.dll, name)
        if name not in _INT_STATUS:
            return fn

        def checked(*args):
            rc = fn(*args)
            if rc != 0:
                msg = self.dll.mq_last_error().decode(errors="replace")
                if rc == MQ_ERR_SAMPLING:
                    raise MQSamplingError(msg)
                raise MQError(f"{name} failed ({rc}): {msg}")
            return rc

        return checked


_LIB = None


def lib() -> _Lib:
    global _LIB
    if _LIB is None:
        _LIB = _Lib(Path(os.environ.get("MQGNN_LIB", LIB_PATH)))
    return _LIB


def ptr(t) -> int | None:
    """Raw device/host address of a torch tensor (None for None)."""
    if t is None:
        return None
    return t.data_ptr()
