"""ctypes binding of the sm_100a library (include/cpsjoin_b200.h).

The product path has no CPU fallback: if the shared library is missing or
no CUDA device is present, every entry point raises.
"""
from __future__ import annotations

import ctypes
import os
import threading

from .build import SO

P = ctypes.c_void_p
i32, i64, u32, u64, dbl = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_double

CPSJ_E_ARG, CPSJ_E_CUDA, CPSJ_E_OOM, CPSJ_E_PICK, CPSJ_E_ABI = -1, -2, -3, -4, -5
ABI_VERSION = (2 << 16) | 0      # CPSJ_ABI_VERSION of include/cpsjoin_b200.h


class _Sized(ctypes.Structure):
    """A parameter struct whose first field is ``struct_size`` (the ABI
    guard of include/cpsjoin_b200.h): filled in automatically, so positional
    construction takes the remaining fields in header order."""

    def __init__(self, *args, **kw):
        super().__init__(ctypes.sizeof(type(self)), *args, **kw)


class Inputs(_Sized):
    _fields_ = [("struct_size", i64), ("d_tokens", P), ("d_offsets", P), ("d_sizes", P), ("n", i64),
                ("d_values", P), ("t", i32), ("d_sketch", P), ("ell", i32), ("d_side", P)]


class Plan(_Sized):
    _fields_ = [("struct_size", i64), ("lambda_", dbl), ("limit", i32), ("depth_cap", i32), ("accept_dist", i32),
                ("flag_dist", i32), ("split_p", dbl), ("h_rep_seeds", P), ("n_reps", i32), ("value_bits", i32),
                ("use_count_table", i32), ("count_threshold", dbl), ("frontier_rank", i32),
                ("frontier_ranks", i32), ("frontier_depth", i32)]


class LshPlan(_Sized):
    _fields_ = [("struct_size", i64), ("lambda_", dbl), ("accept_dist", i32), ("k", i32), ("n_reps", i32),
                ("h_positions", P), ("h_rep_seeds", P), ("cost_only", i32)]


class IngestStats(ctypes.Structure):
    _fields_ = [("n_sets", i64), ("nnz", i64), ("d", i64), ("n_input_records", i64), ("error_line", i64)]


class JoinStats(ctypes.Structure):
    _fields_ = [("n_pairs", i64), ("pre_candidates", i64), ("candidates", i64), ("results", i64),
                ("max_depth", i64), ("peak_live_members", i64), ("n_depth_cap_events", i64),
                ("n_levels", i64), ("gpu_launches", i64), ("lib_calls", i64), ("internal_visits", i64),
                ("split_entries", i64), ("verify_tokens", i64)]


EXPORTS = ["cpsj_version", "cpsj_ctx_create", "cpsj_ctx_destroy", "cpsj_last_error",
           "cpsj_family_create", "cpsj_family_destroy", "cpsj_minhash_sketch", "cpsj_self_join",
           "cpsj_join_copy_result", "cpsj_join_result_device", "cpsj_profile_enable", "cpsj_profile_read",
           "cpsj_launch_counts", "cpsj_frequency_order", "cpsj_exact_join",
           "cpsj_lsh_join", "cpsj_ingest_lists", "cpsj_parse_text", "cpsj_ingest_result_device", "cpsj_ingest_copy",
           "cpsj_minhash_sketch_multi", "cpsj_xbuf_create", "cpsj_xbuf_open", "cpsj_xbuf_close",
           "cpsj_minhash_embed", "cpsj_copy_async", "cpsj_dense_remap"]

MAX_DSTS = 8
IPC_HANDLE_BYTES = 64


class K1Dsts(_Sized):
    _fields_ = [("struct_size", i64), ("d_values", P * MAX_DSTS), ("d_sketch", P * MAX_DSTS), ("n_dsts", i32),
                ("row0", i64)]

PROF_CLASSES = ["k1_minhash", "k4_leaf", "point", "node", "split", "k5_verify", "k6_dedup", "plan"]

_lib = None
_lock = threading.Lock()


class NativeError(RuntimeError):
    pass


def load(path: str | None = None):
    """Load (never build) the shared library; raises if it is absent."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        # CPSJ_LIB: an alternative build of the same sources (A/B diagnostics)
        so = path or os.environ.get("CPSJ_LIB") or SO
        if not os.path.exists(so):
            raise ImportError(f"CUDA library not built: {so} (run python -m paper_1707_06814_b200.build)")
        L = ctypes.CDLL(so)
        L.cpsj_version.restype = ctypes.c_int
        if L.cpsj_version() != ABI_VERSION:
            raise ImportError(f"{so}: ABI version {L.cpsj_version():#x}, this binding expects {ABI_VERSION:#x} "
                              "(rebuild with python -m paper_1707_06814_b200.build)")
        L.cpsj_ctx_create.argtypes = [ctypes.c_int, ctypes.POINTER(P)]
        L.cpsj_ctx_destroy.argtypes = [P]
        L.cpsj_last_error.restype = ctypes.c_char_p
        L.cpsj_last_error.argtypes = [P]
        L.cpsj_family_create.argtypes = [P, P, P, i32, ctypes.POINTER(P)]
        L.cpsj_family_destroy.argtypes = [P]
        L.cpsj_minhash_sketch.argtypes = [P, P, P, P, i64, u32, P, P, P]
        L.cpsj_minhash_embed.argtypes = [P, P, P, P, P, i64, u32, P, P, P]
        L.cpsj_self_join.argtypes = [P, ctypes.POINTER(Inputs), ctypes.POINTER(Plan),
                                     ctypes.POINTER(JoinStats), P]
        L.cpsj_join_copy_result.argtypes = [P, P, P, i64, P, i64, P]
        L.cpsj_join_result_device.argtypes = [P, ctypes.POINTER(P), ctypes.POINTER(P), ctypes.POINTER(i64)]
        L.cpsj_profile_enable.argtypes = [P, ctypes.c_int]
        L.cpsj_profile_read.argtypes = [P, P, P, i32]
        L.cpsj_launch_counts.argtypes = [P, ctypes.POINTER(i64), ctypes.POINTER(i64)]
        L.cpsj_frequency_order.argtypes = [P, P, i64, i64, P, P, P]
        L.cpsj_lsh_join.argtypes = [P, ctypes.POINTER(Inputs), ctypes.POINTER(LshPlan), ctypes.POINTER(JoinStats), P]
        L.cpsj_ingest_lists.argtypes = [P, P, P, i64, i64, ctypes.POINTER(IngestStats), P]
        L.cpsj_parse_text.argtypes = [P, P, i64, i64, ctypes.POINTER(IngestStats), P]
        L.cpsj_ingest_result_device.argtypes = [P, ctypes.POINTER(P), ctypes.POINTER(P), ctypes.POINTER(P)]
        L.cpsj_ingest_copy.argtypes = [P, P, P, P, P]
        L.cpsj_minhash_sketch_multi.argtypes = [P, P, P, P, i64, u32, ctypes.POINTER(K1Dsts), P]
        L.cpsj_xbuf_create.argtypes = [P, i64, ctypes.POINTER(P), P]
        L.cpsj_xbuf_open.argtypes = [P, P, ctypes.POINTER(P)]
        L.cpsj_xbuf_close.argtypes = [P, P, i32]
        L.cpsj_copy_async.argtypes = [P, P, P, i64, P]
        L.cpsj_dense_remap.argtypes = [P, P, i64, i32, P, ctypes.POINTER(i64), P]
        L.cpsj_exact_join.argtypes = [P, P, P, i64, i64, dbl, i32, ctypes.POINTER(JoinStats), P]
        _lib = L
        return L


def check(ctx, rc: int) -> None:
    if rc == 0:
        return
    msg = load().cpsj_last_error(ctx).decode(errors="replace") if ctx else "error"
    if rc == CPSJ_E_ARG:
        raise ValueError(msg)
    if rc == CPSJ_E_ABI:
        raise TypeError(msg)
    if rc == CPSJ_E_PICK:
        raise IndexError(msg)
    if rc == CPSJ_E_OOM:
        raise MemoryError(msg)
    raise NativeError(f"cpsjoin_b200 error {rc}: {msg}")


class Context:
    """One library context per CUDA device."""

    _by_device: dict = {}

    def __init__(self, device: int):
        self.device = device
        self.lib = load()
        h = P()
        check(None, self.lib.cpsj_ctx_create(device, ctypes.byref(h)))
        self.handle = h

    @classmethod
    def get(cls, device: int | None = None) -> "Context":
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("cpsjoin_b200 needs a CUDA device; no CPU fallback exists")
        if device is None:
            device = torch.cuda.current_device()
        ctx = cls._by_device.get(device)
        if ctx is None:
            ctx = cls._by_device[device] = Context(device)
        return ctx

    def check(self, rc: int) -> None:
        check(self.handle, rc)

    def launch_counts(self) -> tuple[int, int]:
        own, lib = i64(), i64()
        self.check(self.lib.cpsj_launch_counts(self.handle, ctypes.byref(own), ctypes.byref(lib)))
        return int(own.value), int(lib.value)

    def profile(self, enable: bool) -> None:
        self.check(self.lib.cpsj_profile_enable(self.handle, int(enable)))

    def profile_read(self) -> dict:
        import numpy as np
        ms = np.zeros(len(PROF_CLASSES), dtype=np.float64)
        cnt = np.zeros(len(PROF_CLASSES), dtype=np.int64)
        self.check(self.lib.cpsj_profile_read(self.handle, ms.ctypes.data, cnt.ctypes.data, len(PROF_CLASSES)))
        return {k: (float(ms[i]), int(cnt[i])) for i, k in enumerate(PROF_CLASSES)}


class Family:
    """A device-resident tabulation-hash family (minhash + optional bit tables)."""

    def __init__(self, ctx: Context, minhash_tables, bit_tables=None):
        import numpy as np
        mh = np.ascontiguousarray(minhash_tables, dtype=np.uint64)
        bt = None if bit_tables is None else np.ascontiguousarray(bit_tables, dtype=np.uint64)
        if mh.ndim != 3 or mh.shape[1:] != (4, 256):
            raise ValueError("tables must have shape (F, 4, 256)")
        self.ctx = ctx
        self.F = mh.shape[0]
        self.has_bits = bt is not None
        h = P()
        ctx.check(ctx.lib.cpsj_family_create(ctx.handle, mh.ctypes.data, None if bt is None else bt.ctypes.data,
                                             self.F, ctypes.byref(h)))
        self.handle = h

    def __del__(self):
        try:
            if getattr(self, "handle", None):
                self.ctx.lib.cpsj_family_destroy(self.handle)
                self.handle = None
        except Exception:
            pass
