"""Dev A/B of the sparse lookup mode on C4-shaped batches (simplex queries and
the acceptance chain queries): FGB_SEARCH_MIXED=1 keeps the bitmap for the
learned path next to the hash for the statistical one."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_00855_b200 import _abi as A, fusegraph as fg, synth  # noqa: E402

docs = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
p = A.synth_params(docs=docs, dense_dim=768, clusters=20, cluster_spread=0.25, learned_vocab=30_522,
                   learned_nnz=120, statistical_vocab=831_592, statistical_nnz=40, entity_vocab=200_000,
                   entity_rate=0.3, max_entities_per_doc=2, kg_triplets=1_000_000, relation_vocab=8,
                   chains=1_000, answers_per_chain=10, seed=1)
c, kg, chains = synth.generate_corpus(p, 0)
dc = fg.DeviceCorpus(c)
ix = fg.build_hybrid_index(dc, kg, degree=32, knn_k=64, knn_iterations=10, seed=42, logical_cap=64)
simplex = synth.synth_queries(p, 10_000, beam_width=608)
dense = np.stack([ch.query_dense for ch in chains])
learned = A.CSR.from_rows([ch.query_learned[0] for ch in chains], [ch.query_learned[1] for ch in chains])
stat = A.CSR.from_rows([ch.query_statistical[0] for ch in chains], [ch.query_statistical[1] for ch in chains])
ents = A.CSR.from_rows([[ch.e0] for ch in chains])
w0 = np.tile(np.array([[1, 1, 1, 0]], np.float32), (len(chains), 1))
chain0 = A.Queries(dense, learned, stat, w0, k=10, beam_width=128, max_entity_hops=2, entities=ents)
for rep in range(2):
    for mixed in ("0", "1"):
        os.environ["FGB_SEARCH_MIXED"] = mixed
        out = []
        for name, q, e in (("simplex", simplex, 512), ("chain_wk0", chain0, 32)):
            fg.batch_query(ix, q, entry_count=e)
            ms = []
            for _ in range(3):
                fg.batch_query(ix, q, entry_count=e)
                ms.append(ix.last_search_stats()[0])
            out.append(f"{name} {q.count / (np.mean(ms) / 1e3):.0f} QPS")
        print(f"mixed={mixed}: " + ", ".join(out), flush=True)
