"""Measurement lines for the SURVEY §8 configs other than the bench's C2, in
the bench.py line format (value / e2e / roofline / cpu_baseline / parity):

  C1  10K docs, d=128, learned + statistical nnz 64 (configs[0]); also the
      reference's build_hybrid_index next to the GPU build
  C3  C2 + statistical vocabulary 831,592, nnz 40 (configs[2]): per-query
      simplex weights over three paths, one index
  C4  C3 + KG: 200K entities, 1M triplets, 1,000 planted 2-hop chains
      (configs[3]); the chain queries of acceptance.cpp:500-511 at 1M docs
      (entities {e0}, 2 hops, beam 128, weights (1,1,1,100) and (1,1,1,0)),
      recall@10 vs the planted answers AND top-k parity vs the reference
  C5  10M docs shaped as C2 (configs[4]) on the GPUs of this box

Same procedure as bench.py: GPU build (upload included), the operating point
selected on a held-out query stream (0x71E6) — the fastest entry x beam
reaching recall@10 0.905 — then recall@10 on the timed batch (stream
0x71E5) against exact GPU truth, the full batch timed on the device (kernel
QPS, L2 flushed) and end to end from pinned host queries.  cpu_baseline: the
UNMODIFIED reference's batch_query (oracle/_ref) over the same index, loaded
from the GPU build's HYBGRIX1 bytes, all host threads, on a bounded sample
whose hits are compared bit for bit with the GPU's.

  python tools/config_bench.py --config C3 [--docs N] [--steps 3]"""
import argparse
import json
import os
import statistics
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2511_00855_b200 import _abi as A, fusegraph as fg, synth  # noqa: E402

CONFIGS = {
    "C1": dict(docs=10_000, dense_dim=128, clusters=20, cluster_spread=0.25, learned_vocab=30_000, learned_nnz=64,
               statistical_vocab=30_000, statistical_nnz=64, seed=1, queries=1_000),
    "C3": dict(docs=1_000_000, dense_dim=768, clusters=20, cluster_spread=0.25, learned_vocab=30_522,
               learned_nnz=120, statistical_vocab=831_592, statistical_nnz=40, seed=1, queries=10_000),
    "C4": dict(docs=1_000_000, dense_dim=768, clusters=20, cluster_spread=0.25, learned_vocab=30_522,
               learned_nnz=120, statistical_vocab=831_592, statistical_nnz=40, entity_vocab=200_000,
               entity_rate=0.3, max_entities_per_doc=2, kg_triplets=1_000_000, relation_vocab=8,
               chains=1_000, answers_per_chain=10, seed=1, queries=10_000),
    "C5": dict(docs=10_000_000, dense_dim=768, clusters=20, cluster_spread=0.25, learned_vocab=30_522,
               learned_nnz=120, statistical_vocab=0, statistical_nnz=0, seed=1, queries=100_000),
}


def timed(ix, q, entry, steps):
    fg.batch_query(ix, q, entry_count=entry)  # warm-up
    kern, wall, launches, r = [], [], 0, None
    for _ in range(steps):
        bench.flush_l2(0)
        t0 = time.perf_counter()
        r = fg.batch_query(ix, q, entry_count=entry)
        wall.append(time.perf_counter() - t0)
        ms, nl = ix.last_search_stats()
        kern.append(ms)
        launches += nl
    return r, kern, wall, launches


def roofline(r, q, kern_ms, R, degree, extra_bytes=0):
    alg = int(r.scored.sum()) * R + int(r.expanded.sum()) * 4 * degree + q.h2d_bytes() + extra_bytes
    ach = alg / (statistics.mean(kern_ms) / 1e3) / 1e9
    peak, kind = bench.peak_hbm()
    return {"bound": "hbm", "achieved": round(ach, 1), "peak": peak, "peak_kind": kind, "unit": "GB/s",
            "frac": round(ach / peak, 4), "traffic": None, "alg_bytes_per_launch": alg,
            "per_query": {"scored": float(r.scored.mean()), "expanded": float(r.expanded.mean()),
                          "row_bytes": R}}


def same_hits(g, rr, m):
    return bool(np.array_equal(g.hit_count[:m], rr.hit_count)
                and np.array_equal(g.doc_id[:m], rr.doc_id)
                and np.array_equal(g.score[:m].view(np.uint64), rr.score.view(np.uint64))
                and np.array_equal(g.expanded[:m], rr.expanded)
                and np.array_equal(g.warnings[:m], rr.warnings))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C3", choices=sorted(CONFIGS))
    ap.add_argument("--docs", type=int, default=0)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--eval-queries", type=int, default=1000)
    ap.add_argument("--cpu-sample", type=int, default=512)
    ap.add_argument("--max-beam", type=int, default=0, help="extend the beam sweep past 2048 (powers of two)")
    ap.add_argument("--no-cpu", action="store_true")
    a = ap.parse_args()
    cfg = dict(CONFIGS[a.config])
    nq = cfg.pop("queries")
    if a.docs:
        cfg["docs"] = a.docs
    p = A.synth_params(**cfg)
    t0 = time.time()
    corpus, kg, chains = synth.generate_corpus(p, 0)
    gen_s = time.time() - t0
    t0 = time.time()
    dc = fg.DeviceCorpus(corpus)
    ix = fg.build_hybrid_index(dc, kg, **bench.BUILD)
    build_s = time.time() - t0
    R = bench.row_bytes(corpus)
    deg = bench.BUILD["degree"]

    held = synth.synth_queries(p, a.eval_queries, stream=bench.HELDOUT_STREAM)
    htruth = fg.brute_force_topk(dc, held)
    if a.max_beam:
        while bench.BEAMS[-1] < a.max_beam:
            bench.BEAMS.append(bench.BEAMS[-1] * 2)
    sweep = bench.sweep_operating_points(fg, ix, held, htruth, a)
    best = bench.select_operating_point(sweep)
    entry, beam = best["entry"], best["beam"]
    queries = synth.synth_queries(p, nq, stream=bench.TIMED_STREAM).with_(beam_width=max(beam, 10))
    ev = queries.subset(np.arange(min(a.eval_queries, nq)))
    truth = fg.brute_force_topk(dc, ev)
    er = fg.batch_query(ix, ev, entry_count=entry)
    recall = float(np.mean([fg.recall_at_k(er.ids(i), truth.ids(i), 10) for i in range(ev.count)]))
    q = queries.pinned()
    r, kern, wall, launches = timed(ix, q, entry, a.steps)
    line = {
        "config": a.config, "metric": bench.METRIC, "unit": "queries/s",
        "value": round(nq / (statistics.mean(kern) / 1e3), 1),
        "e2e": {"value": round(nq / statistics.mean(wall), 1), "unit": "queries/s",
                "h2d_bytes_per_step": int(q.h2d_bytes()), "d2h_bytes_per_step": int(nq * (10 * 20 + 32))},
        "docs": p.docs, "queries": nq, "entry": entry, "beam": beam,
        "recall_at_10": round(recall, 4), "recall_heldout": best["recall"],
        "build_seconds": round(build_s, 2),
        "build_stages_s": {k: round(float(v), 3) for k, v in ix.build_times().items()},
        "gen_seconds": round(gen_s, 1), "gpu_launches": launches,
        "roofline": roofline(r, q, kern, R, deg),
        "operating_point": "held-out sweep (stream 0x71E6), recall on the timed stream 0x71E5",
        "sweep": sweep,
    }
    gpu_chain = {}
    if chains:
        # acceptance.cpp:500-511 at scale
        dense = np.stack([ch.query_dense for ch in chains])
        learned = A.CSR.from_rows([ch.query_learned[0] for ch in chains], [ch.query_learned[1] for ch in chains])
        stat = A.CSR.from_rows([ch.query_statistical[0] for ch in chains],
                               [ch.query_statistical[1] for ch in chains])
        ents = A.CSR.from_rows([[ch.e0] for ch in chains])
        for went in (100.0, 0.0):
            w = np.tile(np.array([[1, 1, 1, went]], np.float32), (len(chains), 1))
            cq = A.Queries(dense, learned, stat, w, k=10, beam_width=128, max_entity_hops=2,
                           entities=ents).pinned()
            cr, ck, cw, cl = timed(ix, cq, 32, a.steps)
            kname = ix.last_search_kernel()
            os.environ["FGB_SEARCH_HYBRID"] = "0"  # A/B: the exact-chain search_kernel
            _, ck0, _, _ = timed(ix, cq, 32, a.steps)
            del os.environ["FGB_SEARCH_HYBRID"]
            rec = float(np.mean([fg.recall_at_k(cr.ids(i), chains[i].answer_docs, 10) for i in range(len(chains))]))
            key = f"chain_queries_wk{int(went)}"
            gpu_chain[key] = (cq, cr)
            line[key] = {
                "queries": len(chains), "beam": 128, "max_entity_hops": 2,
                "recall_at_10_vs_answers": round(rec, 4),
                "value": round(len(chains) / (statistics.mean(ck) / 1e3), 1),
                "e2e": {"value": round(len(chains) / statistics.mean(cw), 1), "unit": "queries/s",
                        "h2d_bytes_per_step": int(cq.h2d_bytes()), "d2h_bytes_per_step": int(len(chains) * 232)},
                "roofline": roofline(cr, cq, ck, R, deg),
                "expanded_per_query": round(float(cr.expanded.mean()), 1),
                "kernel": kname,
                "value_search_kernel": round(len(chains) / (statistics.mean(ck0) / 1e3), 1),
                "queries_with_warnings": int(np.count_nonzero(cr.warnings))}
        line["kg"] = {"triplets": int(len(kg.source)), "chains": len(chains)}

    if p.statistical_vocab:
        # required-keyword queries (keyword_postfilter + twin pool, search.cpp:100-139,
        # 171-181): the first 1,000 timed queries, each requiring its first
        # statistical term (conjunctive)
        kq = queries.subset(np.arange(min(1000, nq)))
        kq.required = A.CSR.from_rows([kq.statistical.row(i)[0][:1].tolist() for i in range(kq.count)])
        kq = kq.pinned()
        kr, kk, kw, kl = timed(ix, kq, entry, a.steps)
        kname = ix.last_search_kernel()
        os.environ["FGB_SEARCH_HYBRID"] = "0"
        _, kk0, _, _ = timed(ix, kq, entry, a.steps)
        del os.environ["FGB_SEARCH_HYBRID"]
        gpu_chain["keyword_queries"] = (kq, kr)
        line["keyword_queries"] = {
            "queries": kq.count, "beam": beam, "entry": entry, "required": "first statistical term, conjunctive",
            "value": round(kq.count / (statistics.mean(kk) / 1e3), 1),
            "e2e": {"value": round(kq.count / statistics.mean(kw), 1), "unit": "queries/s",
                    "h2d_bytes_per_step": int(kq.h2d_bytes()), "d2h_bytes_per_step": int(kq.count * 232)},
            "roofline": roofline(kr, kq, kk, R, deg),
            "kernel": kname,
            "value_search_kernel": round(kq.count / (statistics.mean(kk0) / 1e3), 1),
            "queries_with_shortfall": int(np.count_nonzero(kr.warnings & 2))}
    if not a.no_cpu:
        from oracle.refpy import RefLib, ref_available
        if ref_available():
            ref = RefLib()
            cores = os.cpu_count() or 1
            with tempfile.TemporaryDirectory(prefix="fgb_cfg_") as td:
                path = os.path.join(td, "ix.hyb")
                ix.serialize(path)
                rix = ref.index_deserialize(path)
            m = min(a.cpu_sample, nq)
            sq = queries.subset(np.arange(m))
            pq = ref.prepare_queries(sq)
            t0 = time.perf_counter()
            rr = ref.batch_query_prepared(rix, pq, 0, m, 10, entry_count=entry, threads=cores)
            dt = time.perf_counter() - t0
            line["cpu_baseline"] = {"value": round(m / dt, 2), "unit": "queries/s", "cores": cores,
                                    "cpu_model": bench.cpu_model(), "kind": "reference",
                                    "sample": f"first {m} timed queries, same index (HYBGRIX1 load)"}
            line["parity"] = {"queries": m, "identical": same_hits(r, rr, m)}
            for key, (cq, cr) in gpu_chain.items():
                t0 = time.perf_counter()
                crr = ref.batch_query(rix, cq, entry_count=entry if key == "keyword_queries" else 32,
                                      threads=cores)
                dt = time.perf_counter() - t0
                line[key]["cpu_baseline"] = {"value": round(cq.count / dt, 2), "unit": "queries/s",
                                             "cores": cores, "kind": "reference",
                                             "sample": f"all {cq.count} queries of this set"}
                line[key]["parity"] = {"queries": cq.count, "identical": same_hits(cr, crr, cq.count)}
            if a.config == "C1":
                ix.close()
                dc.close()
                line["build_cpu_baseline"] = bench.build_baseline()
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
