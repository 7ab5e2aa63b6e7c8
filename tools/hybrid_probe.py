"""Dev probe: the hybrid kernel's QPS and exact-resolution counts on
keyword / chain queries vs the same queries as plain batches (C4 shape).

  python tools/hybrid_probe.py [--docs 200000] [--beam 672] [--entry 256]"""
import argparse
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2511_00855_b200 import _abi as A, fusegraph as fg, synth  # noqa: E402
from tools.config_bench import CONFIGS  # noqa: E402


def run(ix, q, entry, label):
    fg.batch_query(ix, q, entry_count=entry)
    ms = []
    for _ in range(3):
        bench.flush_l2(0)
        fg.batch_query(ix, q, entry_count=entry)
        ms.append(ix.last_search_stats()[0])
    print(f"{label:34s} {ix.last_search_kernel():22s} {q.count / (min(ms) / 1e3):10.1f} QPS", flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--docs", type=int, default=200000)
    ap.add_argument("--beam", type=int, default=672)
    ap.add_argument("--entry", type=int, default=256)
    ap.add_argument("--queries", type=int, default=2000)
    a = ap.parse_args()
    cfg = dict(CONFIGS["C4"])
    cfg.pop("queries")
    cfg["docs"] = a.docs
    cfg["chains"] = min(cfg["chains"], a.docs // 1000)
    p = A.synth_params(**cfg)
    c, kg, chains = synth.generate_corpus(p, 0)
    dc = fg.DeviceCorpus(c)
    ix = fg.build_hybrid_index(dc, kg, **bench.BUILD)
    q = synth.synth_queries(p, a.queries, beam_width=a.beam)
    run(ix, q, a.entry, "plain")
    os.environ["FGB_SEARCH_FORCE_HYBRID"] = "1"
    run(ix, q, a.entry, "plain (hybrid kernel)")
    del os.environ["FGB_SEARCH_FORCE_HYBRID"]
    kq = q.subset(np.arange(q.count))
    kq.required = A.CSR.from_rows([kq.statistical.row(i)[0][:1].tolist() for i in range(kq.count)])
    run(ix, kq, a.entry, "keyword")
    os.environ["FGB_SEARCH_TIMING"] = "1"
    fg.batch_query(ix, kq, entry_count=a.entry)
    os.environ["FGB_SEARCH_FORCE_HYBRID"] = "1"
    fg.batch_query(ix, q, entry_count=a.entry)
    del os.environ["FGB_SEARCH_FORCE_HYBRID"]
    del os.environ["FGB_SEARCH_TIMING"]
    os.environ["FGB_SEARCH_STATS"] = "1"
    fg.batch_query(ix, kq, entry_count=a.entry)
    del os.environ["FGB_SEARCH_STATS"]
    os.environ["FGB_SEARCH_HYBRID"] = "0"
    run(ix, kq, a.entry, "keyword (search_kernel)")
    del os.environ["FGB_SEARCH_HYBRID"]
    if chains:
        dense = np.stack([ch.query_dense for ch in chains])
        learned = A.CSR.from_rows([ch.query_learned[0] for ch in chains], [ch.query_learned[1] for ch in chains])
        stat = A.CSR.from_rows([ch.query_statistical[0] for ch in chains], [ch.query_statistical[1] for ch in chains])
        ents = A.CSR.from_rows([[ch.e0] for ch in chains])
        w = np.tile(np.array([[1, 1, 1, 100]], np.float32), (len(chains), 1))
        cq = A.Queries(dense, learned, stat, w, k=10, beam_width=128, max_entity_hops=2, entities=ents)
        run(ix, cq, 32, "chain wk100")
        os.environ["FGB_SEARCH_STATS"] = "1"
        fg.batch_query(ix, cq)
        del os.environ["FGB_SEARCH_STATS"]


if __name__ == "__main__":
    main()
