"""Loader for the in-tree CUDA library libfgb200.so (built by
`make -C paper_2511_00855_b200/csrc` or __graft_entry__.build()).

There is no fallback: if the library is missing or cannot load, importing the
compute API raises.  Every call checks the FG_OK/FG_ERR status and re-raises
the library's error as fgb.Error with the reference's machine code
(error.hpp:11-20)."""
from __future__ import annotations

import ctypes as C
import os

from . import _abi as A

_HERE = os.path.dirname(os.path.abspath(__file__))
# FGB_LIB_VARIANT=x loads libfgb200.x.so (dev A/B builds of the same sources)
_VAR = os.environ.get("FGB_LIB_VARIANT")
LIB_PATH = os.path.join(_HERE, f"libfgb200.{_VAR}.so" if _VAR else "libfgb200.so")


class Error(RuntimeError):
    """Mirror of fusegraph::Error: .code is the machine code, str() is what()."""

    def __init__(self, code: str, what: str):
        super().__init__(what)
        self.code = code


_lib = None


def _declare(lib):
    P = C.POINTER
    sig = {
        "fg_abi_version": (C.c_int, []),
        "fg_last_error_code": (C.c_char_p, []),
        "fg_last_error_message": (C.c_char_p, []),
        "fg_device_count": (C.c_int, [P(C.c_int)]),
        "fg_synth_generate": (C.c_int, [P(A.SynthParams), C.c_uint, P(C.c_void_p)]),
        "fg_host_corpus_view": (C.c_int, [C.c_void_p, P(A.CorpusView), P(A.KgView), A.u64p]),
        "fg_host_corpus_chain": (C.c_int, [C.c_void_p, C.c_uint64, A.u32p, A.u64p, A.u64p, A.f32p,
                                           A.u32p, A.u32p, A.f32p, A.u32p, A.u32p, A.f32p]),
        "fg_host_corpus_free": (C.c_int, [C.c_void_p]),
        "fg_synth_queries": (C.c_int, [P(A.SynthParams), C.c_uint64, C.c_uint64, C.c_int, A.f32p,
                                       A.u32p, A.f32p, A.u32p, A.f32p, P(A.Weights)]),
        "fg_corpus_upload": (C.c_int, [P(A.CorpusView), C.c_int, P(C.c_void_p)]),
        "fg_corpus_free": (C.c_int, [C.c_void_p]),
        "fg_corpus_size": (C.c_int, [C.c_void_p, A.u64p, A.u32p]),
        "fg_corpus_sqnorm": (C.c_int, [C.c_void_p, A.f64p]),
        "fg_corpus_set_deleted": (C.c_int, [C.c_void_p, A.u8p]),
        "fg_build_query_vector": (C.c_int, [P(A.QueryView), C.c_uint64, A.f32p, A.u32p, A.f32p,
                                            A.u32p, A.f32p, A.f64p]),
        "fg_batch_scores": (C.c_int, [C.c_void_p, P(A.QueryView), C.c_uint64, A.u32p, C.c_uint64,
                                      A.f64p]),
        "fg_pair_scores": (C.c_int, [C.c_void_p, A.u32p, A.u32p, C.c_uint64, A.f64p]),
        "fg_knn_init": (C.c_int, [C.c_void_p, C.c_uint32, C.c_uint64, P(A.KnnLists)]),
        "fg_knn_iterate": (C.c_int, [C.c_void_p, P(A.KnnLists), A.u64p]),
        "fg_knn_build": (C.c_int, [C.c_void_p, P(A.KnnParams), P(A.KnnLists), A.u32p]),
        "fg_refine": (C.c_int, [C.c_void_p, P(A.KnnLists), P(A.RefineParams), P(A.Refined),
                                P(A.RefineTrace)]),
        "fg_index_build": (C.c_int, [C.c_void_p, P(A.KgView), P(A.BuildParams), P(C.c_void_p)]),
        "fg_index_create": (C.c_int, [C.c_void_p, P(A.KgView), P(A.GraphView), P(C.c_void_p)]),
        "fg_index_sizes": (C.c_int, [C.c_void_p, A.u32p, A.u64p, A.u64p]),
        "fg_index_export": (C.c_int, [C.c_void_p, A.u32p, A.u64p, A.u32p, A.u64p, A.u32p,
                                      A.u32p]),
        "fg_index_build_times": (C.c_int, [C.c_void_p, A.f64p]),
        "fg_index_build_stats": (C.c_int, [C.c_void_p, A.u64p]),
        "fg_index_build_stats_ex": (C.c_int, [C.c_void_p, A.u64p, C.c_uint32]),
        "fg_index_serialize": (C.c_int, [C.c_void_p, C.c_char_p, A.u64p]),
        "fg_index_insert": (C.c_int, [C.c_void_p, P(A.CorpusView), P(A.InsertParams)]),
        "fg_index_deserialize": (C.c_int, [C.c_char_p, C.c_int, P(C.c_void_p), P(C.c_void_p)]),
        "fg_comm_unique_id": (C.c_int, [A.u8p]),
        "fg_comm_init": (C.c_int, [C.c_int, C.c_int, A.u8p, C.c_int, P(C.c_void_p)]),
        "fg_comm_free": (C.c_int, [C.c_void_p]),
        "fg_comm_init_host": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p,
                                        P(C.c_void_p)]),
        "fg_index_build_sharded": (C.c_int, [C.c_void_p, P(A.KgView), P(A.BuildParams), C.c_void_p,
                                             C.c_uint32, P(C.c_void_p)]),
        "fg_index_free": (C.c_int, [C.c_void_p]),
        "fg_batch_query": (C.c_int, [C.c_void_p, P(A.QueryView), P(A.SearchOpts),
                                     P(A.SearchResults)]),
        "fg_brute_force_topk": (C.c_int, [C.c_void_p, P(A.QueryView), P(A.SearchResults)]),
        "fg_last_search_stats": (C.c_int, [C.c_void_p, A.f64p, A.u64p]),
        "fg_last_search_kernel": (C.c_int, [C.c_void_p, C.POINTER(C.c_char_p)]),
        "fg_refine_tc_stats": (C.c_int, [A.u64p, A.u64p, A.f64p, C.c_int]),
    }
    missing = []
    for name, (res, args) in sig.items():
        fn = getattr(lib, name, None)
        if fn is None:
            missing.append(name)
            continue
        fn.restype = res
        fn.argtypes = args
    lib.fgb_missing = missing
    return lib


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is not built; run `make -C paper_2511_00855_b200/csrc` "
                              "or __graft_entry__.build() (there is no CPU fallback)")
        _lib = _declare(C.CDLL(LIB_PATH))
    return _lib


def check(status: int):
    if status != 0:
        L = lib()
        raise Error(L.fg_last_error_code().decode(), L.fg_last_error_message().decode())


def device_count() -> int:
    n = C.c_int(0)
    check(lib().fg_device_count(C.byref(n)))
    return n.value
