"""Python mirror of the reference's hot-path API (fusegraph::), running on the
B200 through the C-ABI of libfgb200.so (include/fg_b200.h).

Names, argument meaning and error codes follow the reference headers:
  scoring.hpp   -> hybrid_scores / batch_scores / pair_scores
  corpus.hpp    -> build_query_vector
  knn_graph.hpp -> init_random_graph / nn_descent_iterate / build_knn_graph
  refine.hpp    -> refine_graph
  index.hpp     -> build_hybrid_index / HybridIndex.from_graph
  search.hpp    -> batch_query / search
  eval.hpp      -> brute_force_topk / recall_at_k
Every call raises paper_2511_00855_b200.Error(code, what) on failure; there is
no CPU fallback (the library refuses to run without a CUDA device).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _abi as A
from ._lib import Error, check, lib

__all__ = [
    "Error", "DeviceCorpus", "HybridIndex", "build_query_vector", "batch_scores", "pair_scores",
    "init_random_graph", "nn_descent_iterate", "build_knn_graph", "refine_graph",
    "build_hybrid_index", "build_hybrid_index_sharded", "Comm", "batch_query", "search",
    "brute_force_topk", "recall_at_k",
]


class DeviceCorpus:
    """The DocumentStore mirrored in HBM (fg_corpus_upload)."""

    def __init__(self, corpus: A.Corpus, device: int = 0):
        self.host = corpus
        self.n = corpus.n
        self.dense_dim = corpus.dense_dim
        h = C.c_void_p()
        v = corpus.view()
        check(lib().fg_corpus_upload(C.byref(v), device, C.byref(h)))
        self.h = h
        self.device = device

    def close(self):
        if getattr(self, "h", None):
            lib().fg_corpus_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def sqnorm(self) -> np.ndarray:
        out = np.zeros(self.n, np.float64)
        check(lib().fg_corpus_sqnorm(self.h, A.ptr(out, A.f64p)))
        return out

    def set_deleted(self, flags):
        flags = np.ascontiguousarray(flags, np.uint8)
        check(lib().fg_corpus_set_deleted(self.h, A.ptr(flags, A.u8p)))


def build_query_vector(q: A.Queries, i: int):
    """corpus.hpp:34 — (dense, learned_vals, statistical_vals, squared_norm)."""
    dense = np.zeros(q.dense_dim, np.float32)
    li, _ = q.learned.row(i)
    si, _ = q.statistical.row(i)
    lv = np.zeros(max(len(li), 1), np.float32)
    sv = np.zeros(max(len(si), 1), np.float32)
    ln, sn, sq = C.c_uint32(), C.c_uint32(), C.c_double()
    v = q.view()
    check(lib().fg_build_query_vector(C.byref(v), i, A.ptr(dense, A.f32p), C.byref(ln),
                                      A.ptr(lv, A.f32p), C.byref(sn), A.ptr(sv, A.f32p),
                                      C.byref(sq)))
    return dense, lv[:ln.value], sv[:sn.value], sq.value


def batch_scores(dc: DeviceCorpus, q: A.Queries, qi: int, ids) -> np.ndarray:
    """scoring.hpp:32 — hybrid_score of weighted query qi against each id."""
    ids = np.ascontiguousarray(ids, np.uint32)
    out = np.zeros(len(ids), np.float64)
    v = q.view()
    check(lib().fg_batch_scores(dc.h, C.byref(v), qi, A.ptr(ids, A.u32p), len(ids),
                                A.ptr(out, A.f64p)))
    return out


def pair_scores(dc: DeviceCorpus, a, b) -> np.ndarray:
    """hybrid_score(doc a, doc b) under unit weights (knn_graph.cpp:20-22)."""
    a = np.ascontiguousarray(a, np.uint32)
    b = np.ascontiguousarray(b, np.uint32)
    out = np.zeros(len(a), np.float64)
    check(lib().fg_pair_scores(dc.h, A.ptr(a, A.u32p), A.ptr(b, A.u32p), len(a),
                               A.ptr(out, A.f64p)))
    return out


def _lists(n, k):
    return np.zeros((n, k), np.uint32), np.zeros((n, k), np.float64), np.zeros((n, k), np.uint8)


def init_random_graph(dc: DeviceCorpus, k: int, seed: int):
    """knn_graph.hpp:52 — (ids, scores, fresh), each n x k."""
    ids, sc, fr = _lists(dc.n, k)
    s = A.knn_struct(ids, sc, fr)
    check(lib().fg_knn_init(dc.h, k, seed, C.byref(s)))
    return ids, sc, fr


def nn_descent_iterate(dc: DeviceCorpus, ids, sc, fr):
    """knn_graph.hpp:56 — returns (ids, scores, fresh, changed)."""
    ids, sc, fr = (np.ascontiguousarray(x).copy() for x in (ids, sc, fr))
    s = A.knn_struct(ids, sc, fr)
    ch = C.c_uint64()
    check(lib().fg_knn_iterate(dc.h, C.byref(s), C.byref(ch)))
    return ids, sc, fr, ch.value


def build_knn_graph(dc: DeviceCorpus, k=32, max_iterations=12, convergence=0.01, seed=42):
    """knn_graph.hpp:59 — returns (ids, scores, fresh, passes)."""
    kk = min(k, dc.n - 1) if dc.n >= 2 else k
    ids, sc, fr = _lists(dc.n, kk)
    s = A.knn_struct(ids, sc, fr)
    p = A.KnnParams(k, max_iterations, convergence, seed)
    passes = C.c_uint32()
    check(lib().fg_knn_build(dc.h, C.byref(p), C.byref(s), C.byref(passes)))
    return ids, sc, fr, passes.value


def refine_graph(dc: DeviceCorpus, ids, sc, fr, degree=32, per_neighbour=False, trace=False):
    """refine.hpp:87 — (semantic n x degree, keyword [arrays], trace dict|None)."""
    ids, sc, fr = (np.ascontiguousarray(x) for x in (ids, sc, fr))
    n, k = ids.shape
    sem = np.zeros((n, degree), np.uint32)
    kw = np.zeros((n, k), np.uint32)
    kwc = np.zeros(n, np.uint32)
    out = A.Refined(A.ptr(sem, A.u32p), k, A.ptr(kw, A.u32p), A.ptr(kwc, A.u32p))
    t = tr = None
    if trace:
        t = dict(ordered_ids=np.zeros((n, k), np.uint32), ordered_scores=np.zeros((n, k), np.float64),
                 detours=np.zeros((n, k), np.uint32), kept=np.zeros((n, degree), np.uint32),
                 kept_count=np.zeros(n, np.uint32))
        tr = A.RefineTrace(A.ptr(t["ordered_ids"], A.u32p), A.ptr(t["ordered_scores"], A.f64p),
                           A.ptr(t["detours"], A.u32p), A.ptr(t["kept"], A.u32p),
                           A.ptr(t["kept_count"], A.u32p))
    lists = A.knn_struct(ids, sc, fr)
    p = A.RefineParams(degree, int(per_neighbour))
    check(lib().fg_refine(dc.h, C.byref(lists), C.byref(p), C.byref(out),
                          C.byref(tr) if tr is not None else None))
    return sem, [kw[u, :kwc[u]].copy() for u in range(n)], t


class HybridIndex:
    """Device-resident HybridIndex (index.hpp:33-52)."""

    def __init__(self, dc: DeviceCorpus, handle):
        self.corpus = dc
        self.h = handle

    @staticmethod
    def from_graph(dc: DeviceCorpus, graph: dict, kg: A.KG | None = None) -> "HybridIndex":
        """Wrap edge tables built elsewhere (e.g. deserialize_index)."""
        h = C.c_void_p()
        gv = A.graph_view(graph)
        kv = (kg or A.KG()).view()
        check(lib().fg_index_create(dc.h, C.byref(kv), C.byref(gv), C.byref(h)))
        return HybridIndex(dc, h)

    def close(self):
        if getattr(self, "h", None):
            lib().fg_index_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def export(self) -> dict:
        n = self.corpus.n
        deg, kt, lt = C.c_uint32(), C.c_uint64(), C.c_uint64()
        check(lib().fg_index_sizes(self.h, C.byref(deg), C.byref(kt), C.byref(lt)))
        sem = np.zeros((n, deg.value), np.uint32)
        kp = np.zeros(n + 1, np.uint64)
        ki = np.zeros(kt.value, np.uint32)
        lp = np.zeros(n + 1, np.uint64)
        lg = np.zeros((lt.value, 4), np.uint32)
        no = np.zeros(n, np.uint32)
        check(lib().fg_index_export(self.h, A.ptr(sem, A.u32p), A.ptr(kp, A.u64p), A.ptr(ki, A.u32p),
                                    A.ptr(lp, A.u64p), A.ptr(lg, A.u32p), A.ptr(no, A.u32p)))
        return dict(degree=deg.value, semantic=sem, keyword=A.CSR(kp, ki), logical_ptr=lp,
                    logical=lg, norm_order=no)

    def insert(self, docs: A.Corpus, knn_k: int = 0, nn_descent_iterations: int = 10):
        """insert_batch (update.hpp:33): append and link `docs` in place."""
        v = docs.view()
        p = A.InsertParams(knn_k, nn_descent_iterations, 1)
        check(lib().fg_index_insert(self.h, C.byref(v), C.byref(p)))
        n, d = C.c_uint64(), C.c_uint32()
        check(lib().fg_corpus_size(self.corpus.h, C.byref(n), C.byref(d)))
        self.corpus.n = n.value

    def serialize(self, path: str) -> int:
        """serialize_index (io.hpp:63): HYBGRIX1 v1, the reference's bytes."""
        nb = C.c_uint64()
        check(lib().fg_index_serialize(self.h, path.encode(), C.byref(nb)))
        return nb.value

    @staticmethod
    def deserialize(path: str, device: int = 0) -> "HybridIndex":
        """deserialize_index (io.hpp:71) into HBM; the index owns its corpus."""
        ch, ih = C.c_void_p(), C.c_void_p()
        check(lib().fg_index_deserialize(path.encode(), device, C.byref(ch), C.byref(ih)))
        dc = DeviceCorpus.__new__(DeviceCorpus)
        dc.h, dc.device, dc.host = ch, device, None
        n, d = C.c_uint64(), C.c_uint32()
        check(lib().fg_corpus_size(ch, C.byref(n), C.byref(d)))
        dc.n, dc.dense_dim = n.value, d.value
        return HybridIndex(dc, ih)

    def build_times(self) -> dict:
        t = np.zeros(5, np.float64)
        check(lib().fg_index_build_times(self.h, A.ptr(t, A.f64p)))
        return dict(knn=t[0], refine=t[1], logical=t[2], norm_order=t[3], total=t[4])

    def build_stats(self) -> dict:
        t = np.zeros(6, np.uint64)
        check(lib().fg_index_build_stats_ex(self.h, A.ptr(t, A.u64p), 6))
        return dict(passes=int(t[0]), candidates=int(t[1]), dense_rows=int(t[2]), pass_seconds=int(t[3]) / 1e6,
                    sketched=int(t[4]), sketch_rejected=int(t[5]))

    def last_search_stats(self):
        ms, launches = C.c_double(), C.c_uint64()
        check(lib().fg_last_search_stats(self.h, C.byref(ms), C.byref(launches)))
        return ms.value, launches.value

    def last_search_kernel(self) -> str:
        name = C.c_char_p()
        check(lib().fg_last_search_kernel(self.h, C.byref(name)))
        return name.value.decode()


def build_hybrid_index(dc: DeviceCorpus, kg: A.KG | None = None, degree=32, knn_k=32,
                       knn_iterations=10, seed=42, logical_cap=64, default_entity_hops=2,
                       per_neighbour_keyword_check=False) -> HybridIndex:
    """index.hpp:60 — build_hybrid_index on the GPU."""
    h = C.c_void_p()
    p = A.BuildParams(degree, knn_k, knn_iterations, seed, logical_cap, default_entity_hops,
                      int(per_neighbour_keyword_check))
    kv = (kg or A.KG()).view()
    check(lib().fg_index_build(dc.h, C.byref(kv), C.byref(p), C.byref(h)))
    return HybridIndex(dc, h)


class Comm:
    """NCCL communicator of a sharded build (fg_comm_*): one per process/GPU."""

    ID_BYTES = 128

    @staticmethod
    def _torch_nccl_first():
        """The library dlopens libnccl.so.2 on first use; in a PyTorch process
        that must resolve to the NCCL torch bundles (once a libnccl.so.2 is
        loaded, torch's own can no longer be)."""
        import torch  # noqa: F401  (loads torch's libnccl)

    @staticmethod
    def unique_id() -> bytes:
        Comm._torch_nccl_first()
        buf = np.zeros(Comm.ID_BYTES, np.uint8)
        check(lib().fg_comm_unique_id(A.ptr(buf, A.u8p)))
        return buf.tobytes()

    def __init__(self, nranks: int, rank: int, uid: bytes, device: int = 0):
        Comm._torch_nccl_first()
        buf = np.frombuffer(uid, np.uint8).copy()
        h = C.c_void_p()
        check(lib().fg_comm_init(nranks, rank, A.ptr(buf, A.u8p), device, C.byref(h)))
        self.h, self.rank, self.size = h, rank, nranks

    def close(self):
        if getattr(self, "h", None):
            lib().fg_comm_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_HOST_GATHER = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64)
_HOST_SUM = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_uint64), C.c_uint64)


class HostComm(Comm):
    """A sharded-build communicator whose collectives run on host buffers
    through torch.distributed (fg_comm_init_host) — any backend, e.g. gloo.
    Lets several ranks share one GPU (NCCL refuses that), so the multi-rank
    build is exercised by multi-process tests on a single-GPU box."""

    def __init__(self, nranks: int, rank: int, device: int = 0):
        import torch
        import torch.distributed as dist

        def gather(_ctx, send, recv, nbytes):
            try:
                src = np.ctypeslib.as_array((C.c_uint8 * nbytes).from_address(send)).copy()
                parts = [torch.empty(nbytes, dtype=torch.uint8) for _ in range(nranks)]
                dist.all_gather(parts, torch.from_numpy(src))
                dst = np.ctypeslib.as_array((C.c_uint8 * (nbytes * nranks)).from_address(recv))
                dst[:] = torch.cat(parts).numpy()
                return 0
            except Exception:  # reported to the library as a failed collective
                return 1

        def total(_ctx, x, count):
            try:
                t = torch.tensor([int(x[i]) for i in range(count)], dtype=torch.int64)
                dist.all_reduce(t)
                for i in range(count):
                    x[i] = int(t[i])
                return 0
            except Exception:
                return 1

        self._cb = (_HOST_GATHER(gather), _HOST_SUM(total))  # kept alive with the comm
        h = C.c_void_p()
        check(lib().fg_comm_init_host(nranks, rank, device, C.cast(self._cb[0], C.c_void_p),
                                      C.cast(self._cb[1], C.c_void_p), None, C.byref(h)))
        self.h, self.rank, self.size = h, rank, nranks


def build_hybrid_index_sharded(dc: DeviceCorpus, kg: A.KG | None = None, comm: Comm | None = None,
                               sim_ranks: int = 1, degree=32, knn_k=32, knn_iterations=10, seed=42,
                               logical_cap=64, default_entity_hops=2,
                               per_neighbour_keyword_check=False) -> HybridIndex:
    """build_hybrid_index sharded by vertex range over `comm`'s
    ranks (one GPU each, NCCL all-gathers), or — comm None — over `sim_ranks`
    ranges computed in this process.  Identical to build_hybrid_index."""
    h = C.c_void_p()
    p = A.BuildParams(degree, knn_k, knn_iterations, seed, logical_cap, default_entity_hops,
                      int(per_neighbour_keyword_check))
    kv = (kg or A.KG()).view()
    check(lib().fg_index_build_sharded(dc.h, C.byref(kv), C.byref(p), comm.h if comm else None,
                                       sim_ranks, C.byref(h)))
    return HybridIndex(dc, h)


def batch_query(ix: HybridIndex, q: A.Queries, entry_count=32, conjunctive=True) -> A.Results:
    """search.hpp:86 — one result row per query; per-query errors captured."""
    res = A.Results(q.count, int(q.k.max()) if q.count else 1)
    rs = res.struct()
    v = q.view()
    o = A.SearchOpts(entry_count, int(conjunctive))
    check(lib().fg_batch_query(ix.h, C.byref(v), C.byref(o), C.byref(rs)))
    return res


def search(ix: HybridIndex, q: A.Queries, i: int = 0, entry_count=32, conjunctive=True):
    """search.hpp:84 — single query; raises on a validation error like search()."""
    sub = q.subset([i])
    res = batch_query(ix, sub, entry_count, conjunctive)
    err = res.error(0)
    if err:
        raise Error(err.split(":", 1)[0], err)
    return res


def brute_force_topk(dc: DeviceCorpus, q: A.Queries) -> A.Results:
    """eval.hpp:20 — exhaustive truth for every query."""
    res = A.Results(q.count, int(q.k.max()) if q.count else 1)
    rs = res.struct()
    v = q.view()
    check(lib().fg_brute_force_topk(dc.h, C.byref(v), C.byref(rs)))
    return res


def recall_at_k(result, truth, k: int) -> float:
    """eval.cpp:53-63."""
    if k == 0:
        raise Error("invalid-k", "invalid-k: recall@k needs k > 0")
    t = set(int(x) for x in truth)
    hits = sum(1 for x in list(result)[:k] if int(x) in t)
    return hits / k


def refine_tc_stats(reset: bool = True) -> dict:
    """Counters of the refinery's tensor-core Gram (fg_refine_tc_stats)."""
    pairs, res, mx = C.c_uint64(), C.c_uint64(), C.c_double()
    check(lib().fg_refine_tc_stats(C.byref(pairs), C.byref(res), C.byref(mx), int(reset)))
    return {"pairs": pairs.value, "resolved": res.value, "max_rel_err": mx.value}
