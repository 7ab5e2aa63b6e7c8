"""Measurement lines for the SURVEY §8 configs other than the bench's C2:
C1 (10K docs, d=128, learned + statistical nnz 64), C3 (C2 + statistical
vocabulary 831,592, nnz 40: the statistical path takes the hash lookups),
C4 (C3 + KG: 200K entities, 1M triplets, 1,000 planted 2-hop chains; the
chain queries of acceptance.cpp:500-511 at 1M docs) and C5 (10M docs shaped
as C2 on ONE GPU: this box has one B200, so the 2/4/8-GPU sharding of C5 is
covered by the simulated-rank parity tests, not measured here).
Same procedure as bench.py: GPU build, exact GPU truth on 1,000 queries, the
entry x beam sweep to recall@10 >= 0.9, then the full batch timed on the
device (kernel QPS) and end to end from pinned host queries.
  python tools/config_bench.py --config C3 [--docs N] [--steps 3]"""
import argparse
import json
import os
import statistics
import sys
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

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C3", choices=sorted(CONFIGS))
ap.add_argument("--docs", type=int, default=0)
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--eval-queries", type=int, default=1000)
ap.add_argument("--max-beam", type=int, default=0, help="extend the beam sweep past 2048 (powers of two)")
a = ap.parse_args()
cfg = dict(CONFIGS[a.config])
nq = cfg.pop("queries")
if a.docs:
    cfg["docs"] = a.docs
p = A.synth_params(**cfg)
t0 = time.time()
corpus, kg, chains = synth.generate_corpus(p, 0)
gen_s = time.time() - t0
dc = fg.DeviceCorpus(corpus)
t0 = time.time()
ix = fg.build_hybrid_index(dc, kg, **bench.BUILD)
build_s = time.time() - t0
queries = synth.synth_queries(p, nq)
ev = queries.subset(np.arange(min(a.eval_queries, nq)))
truth = fg.brute_force_topk(dc, ev)
if a.max_beam:
    while bench.BEAMS[-1] < a.max_beam:
        bench.BEAMS.append(bench.BEAMS[-1] * 2)
sweep = bench.sweep_operating_points(fg, ix, ev, truth, argparse.Namespace(entry=0, beam=0))
best = bench.select_operating_point(sweep)
q = queries.with_(beam_width=max(best["beam"], 10)).pinned()
fg.batch_query(ix, q, entry_count=best["entry"])  # warm-up
kern, wall = [], []
for _ in range(a.steps):
    bench.flush_l2(0)
    t0 = time.perf_counter()
    r = fg.batch_query(ix, q, entry_count=best["entry"])
    wall.append(time.perf_counter() - t0)
    kern.append(ix.last_search_stats()[0])
extra = {}
if chains:
    # acceptance.cpp:500-511 at scale: vector = chain.query_vector, entities {e0},
    # k 10, beam 128, max_entity_hops 2, weights (1,1,1,100) vs (1,1,1,0);
    # recall@10 against the chain's planted answer docs
    dense = np.stack([ch.query_dense for ch in chains])
    learned = A.CSR.from_rows([ch.query_learned[0] for ch in chains], [ch.query_learned[1] for ch in chains])
    stat = A.CSR.from_rows([ch.query_statistical[0] for ch in chains],
                           [ch.query_statistical[1] for ch in chains])
    ents = A.CSR.from_rows([[ch.e0] for ch in chains])
    for went in (100.0, 0.0):
        w = np.tile(np.array([[1, 1, 1, went]], np.float32), (len(chains), 1))
        cq = A.Queries(dense, learned, stat, w, k=10, beam_width=128, max_entity_hops=2, entities=ents).pinned()
        fg.batch_query(ix, cq)
        ck, cw = [], []
        for _ in range(a.steps):
            bench.flush_l2(0)
            t0 = time.perf_counter()
            cr = fg.batch_query(ix, cq)
            cw.append(time.perf_counter() - t0)
            ck.append(ix.last_search_stats()[0])
        rec = float(np.mean([fg.recall_at_k(cr.ids(i), chains[i].answer_docs, 10) for i in range(len(chains))]))
        extra[f"chain_queries_wk{int(went)}"] = {
            "queries": len(chains), "beam": 128, "max_entity_hops": 2, "recall_at_10_vs_answers": round(rec, 4),
            "qps_kernel": round(len(chains) / (statistics.mean(ck) / 1e3), 1),
            "qps_e2e": round(len(chains) / statistics.mean(cw), 1),
            "expanded_per_query": round(float(cr.expanded.mean()), 1),
            "queries_with_warnings": int(np.count_nonzero(cr.warnings))}
    extra["kg"] = {"triplets": int(len(kg.source)), "chains": len(chains)}
print(json.dumps({
    "config": a.config, "docs": p.docs, "queries": nq, "entry": best["entry"], "beam": best["beam"],
    "recall_at_10": best["recall"], "qps_kernel": round(nq / (statistics.mean(kern) / 1e3), 1),
    "qps_e2e": round(nq / statistics.mean(wall), 1), "build_s": round(build_s, 2),
    "build_stages_s": {k: round(float(v), 3) for k, v in ix.build_times().items()}, "gen_s": round(gen_s, 1),
    "scored_per_query": round(float(r.scored.mean()), 1), "expanded_per_query": round(float(r.expanded.mean()), 1),
    "sweep": sweep, **extra}), flush=True)
