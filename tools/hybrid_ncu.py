"""Profiling driver for search_hybrid_kernel at the C4 shape: chain queries
(acceptance.cpp:500-511 shape, w_k = 100) twice, then required-keyword
queries twice; run under
  ncu -k regex:search_hybrid -s 1 -c 3 ...
to capture the second chain batch and both keyword batches."""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2511_00855_b200 import _abi as A, fusegraph as fg, synth  # noqa: E402
from tools.config_bench import CONFIGS  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--docs", type=int, default=1_000_000)
ap.add_argument("--queries", type=int, default=10_000)
a = ap.parse_args()
cfg = dict(CONFIGS["C4"])
cfg.pop("queries")
cfg["docs"] = a.docs
p = A.synth_params(**cfg)
c, kg, chains = synth.generate_corpus(p, 0)
dc = fg.DeviceCorpus(c)
ix = fg.build_hybrid_index(dc, kg, **bench.BUILD)
dense = np.stack([ch.query_dense for ch in chains])
learned = A.CSR.from_rows([ch.query_learned[0] for ch in chains], [ch.query_learned[1] for ch in chains])
stat = A.CSR.from_rows([ch.query_statistical[0] for ch in chains], [ch.query_statistical[1] for ch in chains])
w = np.tile(np.array([[1, 1, 1, 100]], np.float32), (len(chains), 1))
cq = A.Queries(dense, learned, stat, w, k=10, beam_width=128, max_entity_hops=2,
               entities=A.CSR.from_rows([[ch.e0] for ch in chains]))
for _ in range(2):
    fg.batch_query(ix, cq)
    print("chain", ix.last_search_kernel(), len(chains) / (ix.last_search_stats()[0] / 1e3), flush=True)
q = synth.synth_queries(p, a.queries, beam_width=672)
q.required = A.CSR.from_rows([q.statistical.row(i)[0][:1].tolist() for i in range(q.count)])
for _ in range(2):
    fg.batch_query(ix, q, entry_count=512)
    print("keyword", ix.last_search_kernel(), q.count / (ix.last_search_stats()[0] / 1e3), flush=True)
