"""ctypes declarations of include/qsim.h.  Loads the in-tree libqsim_b200.so
and fails loudly if it is missing: there is no CPU fallback."""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("QSIM_LIB") or os.path.join(HERE, "libqsim_b200.so")

QSIM_MAX_CONTROLS = 8
QSIM_MAX_PERM_TARGETS = 12
TRANSPORT_LOCAL, TRANSPORT_VIRTUAL, TRANSPORT_NCCL, TRANSPORT_LOOPBACK = 0, 1, 2, 3

STATUS = ["QSIM_OK", "QSIM_ERR_ARG", "QSIM_ERR_QUBIT_RANGE", "QSIM_ERR_DUP_QUBIT", "QSIM_ERR_NOT_UNITARY",
          "QSIM_ERR_NOT_PERMUTATION", "QSIM_ERR_OOM", "QSIM_ERR_CUDA", "QSIM_ERR_COMM", "QSIM_ERR_STATE",
          "QSIM_ERR_UNSUPPORTED"]


class c128(ctypes.Structure):
    _fields_ = [("re", ctypes.c_double), ("im", ctypes.c_double)]


class qsim_gate(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("target", ctypes.c_int32), ("n_controls", ctypes.c_int32),
                ("n_targets", ctypes.c_int32), ("controls", ctypes.c_int32 * QSIM_MAX_CONTROLS),
                ("targets", ctypes.c_int32 * QSIM_MAX_PERM_TARGETS), ("u", c128 * 4),
                ("perm", ctypes.POINTER(ctypes.c_uint32))]


class qsim_config(ctypes.Structure):
    _fields_ = [("n_qubits", ctypes.c_int32), ("n_ranks", ctypes.c_int32), ("rank", ctypes.c_int32),
                ("transport", ctypes.c_int32), ("shards", ctypes.c_void_p * 64), ("scratch", ctypes.c_void_p),
                ("scratch_bytes", ctypes.c_size_t), ("stream", ctypes.c_void_p),
                ("nccl_id", ctypes.c_uint8 * 128)]


class qsim_stats(ctypes.Structure):
    _fields_ = [(k, ctypes.c_uint64) for k in ("gates", "flushes", "passes", "generic_launches", "perm_launches",
                                              "exchanges", "exchange_bytes", "kernel_launches", "relabels")] + \
               [(k, ctypes.c_double) for k in ("pass_ms", "generic_ms", "perm_ms", "exchange_ms", "reduce_ms",
                                              "plan_ms")] + [("pass_amp_bytes", ctypes.c_uint64),
                                                            ("jit_launches", ctypes.c_uint64),
                                                            ("jit_kernels", ctypes.c_uint64),
                                                            ("jit_compile_ms", ctypes.c_double),
                                                            ("pass_fp64_slots", ctypes.c_double),
                                                            ("plan_cache_hits", ctypes.c_uint64),
                                                            ("streamed_steps", ctypes.c_uint64),
                                                            ("overlapped", ctypes.c_uint64),
                                                            ("overlap_ms", ctypes.c_double),
                                                            ("link_gbs", ctypes.c_double),
                                                            ("fused_readouts", ctypes.c_uint64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


EXPORTS = [
    "qsim_create", "qsim_create_ext", "qsim_create_rank", "qsim_scratch_bytes", "qsim_get_unique_id",
    "qsim_get_loopback_id", "qsim_destroy",
    "qsim_init_basis", "qsim_apply_1q", "qsim_apply_controlled", "qsim_apply_perm", "qsim_apply_swap",
    "qsim_remap", "qsim_run_circuit", "qsim_probabilities", "qsim_expectations", "qsim_expectations_async",
    "qsim_measure",
    "qsim_get_amplitudes", "qsim_sync", "qsim_get_layout", "qsim_set_option", "qsim_get_stats",
    "qsim_reset_stats", "qsim_status_str", "qsim_last_error", "qsim_plan_json", "qsim_exchange_peers",
    "qsim_probe_peaks",
]

_lib = None


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with __graft_entry__.build() "
                          "(python -m paper_quant_ph_0608239_b200.build); there is no CPU fallback")
    L = ctypes.CDLL(LIB_PATH)
    P = ctypes.POINTER
    ctx = ctypes.c_void_p
    i, u64, d, st = ctypes.c_int, ctypes.c_uint64, ctypes.c_double, ctypes.c_int
    sig = {
        "qsim_create": ([i, i, P(ctx)], st),
        "qsim_create_ext": ([P(qsim_config), P(ctx)], st),
        "qsim_create_rank": ([i, i, i, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p,
                              ctypes.c_size_t, ctypes.c_void_p, P(ctx)], st),
        "qsim_scratch_bytes": ([i, i], ctypes.c_size_t),
        "qsim_get_unique_id": ([ctypes.c_void_p], st),
        "qsim_get_loopback_id": ([ctypes.c_void_p], st),
        "qsim_destroy": ([ctx], st),
        "qsim_init_basis": ([ctx, u64], st),
        "qsim_apply_1q": ([ctx, i, P(c128)], st),
        "qsim_apply_controlled": ([ctx, P(i), i, i, P(c128)], st),
        "qsim_apply_perm": ([ctx, P(i), i, P(i), i, P(ctypes.c_uint32)], st),
        "qsim_apply_swap": ([ctx, i, i], st),
        "qsim_remap": ([ctx, P(i), P(i), i], st),
        "qsim_run_circuit": ([ctx, P(qsim_gate), ctypes.c_size_t], st),
        "qsim_probabilities": ([ctx, P(i), i, P(d)], st),
        "qsim_expectations": ([ctx, P(d)], st),
        "qsim_expectations_async": ([ctx, ctypes.c_void_p], st),
        "qsim_measure": ([ctx, P(i), i, u64, u64, P(u64)], st),
        "qsim_get_amplitudes": ([ctx, u64, u64, P(c128)], st),
        "qsim_sync": ([ctx], st),
        "qsim_get_layout": ([ctx, P(i)], st),
        "qsim_set_option": ([ctx, ctypes.c_char_p, ctypes.c_int64], st),
        "qsim_get_stats": ([ctx, P(qsim_stats)], st),
        "qsim_reset_stats": ([ctx], st),
        "qsim_status_str": ([st], ctypes.c_char_p),
        "qsim_last_error": ([ctx], ctypes.c_char_p),
        "qsim_plan_json": ([i, i, P(qsim_gate), ctypes.c_size_t, i, ctypes.c_char_p, ctypes.c_size_t], st),
        "qsim_exchange_peers": ([i, i, i, P(i), i, P(i), P(i)], st),
        "qsim_probe_peaks": ([P(d), P(d)], st),
    }
    for name, (args, res) in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    _lib = L
    return L
