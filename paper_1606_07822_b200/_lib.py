"""ctypes binding of libcachegram_b200.so (the C-ABI in include/cachegram_b200.h).

The shared library is built in-tree by ``__graft_entry__.build()`` (nvcc, sm_100a).
Loading fails loudly when it is missing: there is no Python or CPU fallback for
any training computation.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

PKG_DIR = Path(__file__).resolve().parent
# CG_LIB: an alternative build of the same library (tools/ab_build.py, same-box A/B
# timing of kernel variants); unset in every test, smoke and bench run.
LIB_PATH = Path(os.environ["CG_LIB"]) if os.environ.get("CG_LIB") else PKG_DIR / "libcachegram_b200.so"

CG_OK = 0
CG_ERR_INVALID_ARGUMENT = 1
CG_ERR_IO = 2
CG_ERR_CUDA = 3
CG_ERR_NCCL = 4
CG_ERR_NO_TRAINABLE_WORDS = 5
CG_ERR_INTERNAL = 6
CG_ERR_PARSE = 7

CG_FORMAT_TEXT = 0
CG_FORMAT_BINARY = 1
CG_FORMAT_AUTO = 2

CG_MODE_HOGWILD = 0
CG_MODE_DETERMINISTIC = 1


class CgConfig(C.Structure):
    _fields_ = [
        ("dim", C.c_int32),
        ("window", C.c_int32),
        ("min_count", C.c_int64),
        ("sample", C.c_double),
        ("alpha0", C.c_float),
        ("iterations", C.c_int32),
        ("workers", C.c_int32),
        ("cache_nodes", C.c_int32),
        ("flush_interval", C.c_int32),
        ("seed", C.c_uint64),
    ]


class CgModelDesc(C.Structure):
    _fields_ = [
        ("vocab_size", C.c_int32),
        ("counts", C.POINTER(C.c_int64)),
        ("total_tokens", C.c_int64),
        ("path_offsets", C.POINTER(C.c_int64)),
        ("path_nodes", C.POINTER(C.c_int32)),
        ("path_turns", C.POINTER(C.c_uint8)),
        ("node_usage", C.POINTER(C.c_int64)),
        ("hot_nodes", C.POINTER(C.c_int32)),
        ("hot_count", C.c_int32),
    ]


class CgTrainStats(C.Structure):
    _fields_ = [
        ("words_processed", C.c_uint64),
        ("wall_seconds", C.c_double),
        ("words_per_second", C.c_double),
        ("kernel_seconds", C.c_double),
        ("centers", C.c_uint64),
        ("pairs", C.c_uint64),
        ("steps", C.c_uint64),
    ]


class CgEpochStats(C.Structure):
    _fields_ = [
        ("words", C.c_uint64),
        ("kept", C.c_uint64),
        ("pairs", C.c_uint64),
        ("steps", C.c_uint64),
        ("train_ms", C.c_double),
        ("subsample_ms", C.c_double),
        ("train_launches", C.c_int32),
        ("other_launches", C.c_int32),
        ("cached_rows", C.c_int32),
        ("worker_warps", C.c_int32),
        ("ctx_batch", C.c_int32),
        ("blocks", C.c_int32),
        ("smem_rows", C.c_int32),
        ("floor_rows", C.c_int32),
        ("flush_centers", C.c_int32),
        ("kernel", C.c_int32),
    ]


class CgTuning(C.Structure):
    _fields_ = [("blocks", C.c_int32), ("warps_per_block", C.c_int32), ("centers_per_warp", C.c_int32),
                ("smem_cache_rows", C.c_int32), ("hot_flush_scale", C.c_float), ("flush_centers", C.c_int32),
                ("min_cache_rows", C.c_int32), ("kernel", C.c_int32)]


P = C.POINTER
vp = C.c_void_p
SIGMOID_FN = C.CFUNCTYPE(C.c_float, C.c_float, C.c_void_p)
# name -> (restype, argtypes); mirrors include/cachegram_b200.h
SIGNATURES = {
    "cg_abi_version": (C.c_int, []),
    "cg_last_error": (C.c_char_p, []),
    "cg_device_count": (C.c_int, []),
    "cg_release_cached_memory": (None, []),
    "cg_keep_probability": (C.c_double, [C.c_int64, C.c_int64, C.c_double]),
    "cg_update_alpha": (C.c_float, [C.c_uint64, C.c_uint64, C.c_float]),
    "cg_sigmoid_table": (None, [P(C.c_float)]),
    "cg_init_model": (C.c_int, [C.c_int32, C.c_int32, C.c_uint64, P(C.c_float)]),
    "cg_build_huffman": (C.c_int, [P(C.c_int64), C.c_int32, P(C.c_int64), P(C.c_int32), P(C.c_uint8),
                                   P(C.c_int64), P(C.c_int64)]),
    "cg_select_cached_nodes": (C.c_int32, [P(C.c_int64), C.c_int32, C.c_int32, P(C.c_int32), P(C.c_int32)]),
    "cg_corpus_open": (C.c_int, [C.c_char_p, C.c_int64, P(vp)]),
    "cg_corpus_vocab_size": (C.c_int32, [vp]),
    "cg_corpus_total_tokens": (C.c_int64, [vp]),
    "cg_corpus_word_bytes": (C.c_int64, [vp]),
    "cg_corpus_export_vocab": (C.c_int, [vp, P(C.c_int64), C.c_char_p]),
    "cg_corpus_read_ids": (C.c_int, [vp, C.c_char_p, P(C.c_int32), C.c_int64, P(C.c_int64)]),
    "cg_corpus_close": (None, [vp]),
    "cg_train": (C.c_int, [P(CgConfig), C.c_int32, P(CgModelDesc), P(C.c_int32), C.c_int64, P(C.c_float),
                           P(C.c_float), P(CgTrainStats)]),
    "cg_train_center": (C.c_int, [C.c_int32, P(C.c_int32), C.c_int64, C.c_int64, C.c_int32, C.c_int32, C.c_int32,
                                  P(C.c_float), P(C.c_float), P(C.c_int64), P(C.c_int32), P(C.c_uint8),
                                  P(C.c_int32), C.c_int32, P(C.c_float), P(C.c_float), P(C.c_uint8), C.c_float,
                                  C.c_int32, C.c_float, P(C.c_int64)]),
    "cg_train_center_cb": (C.c_int, [C.c_int32, P(C.c_int32), C.c_int64, C.c_int64, C.c_int32, C.c_int32, C.c_int32,
                                     P(C.c_float), P(C.c_float), P(C.c_int64), P(C.c_int32), P(C.c_uint8),
                                     P(C.c_int32), C.c_int32, P(C.c_float), P(C.c_float), P(C.c_uint8), C.c_float,
                                     C.c_void_p, C.c_void_p, P(C.c_int64)]),
    "cg_cache_flush": (C.c_int, [C.c_int32, C.c_int32, P(C.c_float), P(C.c_int32), C.c_int32, P(C.c_float),
                                 P(C.c_float), P(C.c_uint8)]),
    "cg_session_create": (C.c_int, [P(CgConfig), C.c_int32, P(CgModelDesc), C.c_int32, vp, P(vp)]),
    "cg_session_destroy": (None, [vp]),
    "cg_session_upload_ids": (C.c_int, [vp, P(C.c_int32), C.c_int64]),
    "cg_session_upload_ids_device": (C.c_int, [vp, vp, C.c_int64]),
    "cg_session_reset_model": (C.c_int, [vp]),
    "cg_session_set_model": (C.c_int, [vp, P(C.c_float), P(C.c_float)]),
    "cg_session_train_range": (C.c_int, [vp, C.c_int32, C.c_int64, C.c_int64, C.c_uint64, C.c_uint32,
                                         P(CgEpochStats)]),
    "cg_session_train": (C.c_int, [vp, P(CgTrainStats)]),
    "cg_session_download": (C.c_int, [vp, P(C.c_float), P(C.c_float)]),
    "cg_session_model_buffer": (C.c_int, [vp, P(vp), P(C.c_size_t), P(C.c_int32)]),
    "cg_session_tune": (C.c_int, [vp, P(CgTuning)]),
    "cg_session_sync_begin": (C.c_int, [vp]),
    "cg_session_sync_delta": (C.c_int, [vp, P(vp), P(C.c_size_t)]),
    "cg_session_sync_apply": (C.c_int, [vp, C.c_int32, C.c_uint64]),
    "cg_sync_row_scale": (C.c_float, [C.c_double, C.c_int32, C.c_double]),
    "cg_corpus_open_gpu": (C.c_int, [C.c_char_p, C.c_int64, C.c_int32, P(vp)]),
    "cg_corpus_read_ids_gpu": (C.c_int, [vp, C.c_char_p, C.c_int32, P(C.c_int32), C.c_int64, P(C.c_int64)]),
    "cg_session_load_corpus": (C.c_int, [vp, C.c_char_p, C.c_char_p, P(C.c_int64)]),
    "cg_train_file": (C.c_int, [P(CgConfig), C.c_int32, P(CgModelDesc), C.c_char_p, C.c_char_p, P(C.c_float),
                                P(C.c_float), P(CgTrainStats)]),
    "cg_train_replicas": (C.c_int, [P(CgConfig), C.c_int32, P(CgModelDesc), P(C.c_int32), C.c_int64, P(C.c_int32),
                                    C.c_int32, C.c_int64, P(C.c_float), P(C.c_float), P(CgTrainStats)]),
    "cg_train_file_replicas": (C.c_int, [P(CgConfig), C.c_int32, P(CgModelDesc), C.c_char_p, C.c_char_p,
                                         P(C.c_int32), C.c_int32, C.c_int64, P(C.c_float), P(C.c_float),
                                         P(CgTrainStats)]),
    "cg_average_buffers": (C.c_int, [P(vp), P(C.c_int32), C.c_int32, C.c_size_t]),
    "cg_embeddings_create": (C.c_int, [P(C.c_float), C.c_int32, C.c_int32, C.c_int32, P(vp)]),
    "cg_embeddings_create_device": (C.c_int, [vp, C.c_int32, C.c_int32, C.c_int32, C.c_int32, P(vp)]),
    "cg_embeddings_destroy": (None, [vp]),
    "cg_embeddings_rows": (C.c_int32, [vp]),
    "cg_embeddings_normalized": (C.c_int, [vp, P(C.c_float)]),
    "cg_analogy_answer": (C.c_int, [vp, P(C.c_int32), C.c_int64, P(C.c_int32)]),
    "cg_nearest": (C.c_int, [vp, P(C.c_int32), C.c_int64, C.c_int32, P(C.c_int32), P(C.c_float)]),
    "cg_model_save": (C.c_int, [C.c_char_p, C.c_int32, C.c_char_p, P(C.c_float), C.c_int32, C.c_int32]),
    "cg_model_load": (C.c_int, [C.c_char_p, C.c_int32, P(vp)]),
    "cg_model_file_info": (C.c_int, [vp, P(C.c_int32), P(C.c_int32), P(C.c_int64)]),
    "cg_model_file_export": (C.c_int, [vp, C.c_char_p, P(C.c_float)]),
    "cg_model_file_close": (None, [vp]),
}

_lib = None


def load() -> C.CDLL:
    """Load the CUDA library; raises if it has not been built (no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise RuntimeError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(the GPU path has no CPU fallback)")
    lib = C.CDLL(str(LIB_PATH), mode=os.RTLD_NOW | os.RTLD_LOCAL)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def exported_symbols() -> list[str]:
    return list(SIGNATURES)


class ParseError(RuntimeError):
    """A model or question file violates its format (the reference's ParseError)."""


class CgError(RuntimeError):
    def __init__(self, code: int, message: str):
        super().__init__(message)
        self.code = code


def check(rc: int) -> None:
    if rc != CG_OK:
        msg = load().cg_last_error().decode("utf-8", "replace")
        if rc == CG_ERR_INVALID_ARGUMENT:
            raise ValueError(msg)
        if rc == CG_ERR_IO:
            raise OSError(msg)
        if rc == CG_ERR_PARSE:
            raise ParseError(msg)
        raise CgError(rc, msg)


def ptr(a: np.ndarray | None, ctype):
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"], "arrays crossing the C-ABI must be contiguous"
    return a.ctypes.data_as(C.POINTER(ctype))
