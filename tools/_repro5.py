import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_2511_00855_b200 import _abi as A, fusegraph as fg, synth
p = A.synth_params(docs=1500, entity_vocab=40, kg_triplets=150, chains=50, answers_per_chain=10, seed=51)
c, kg, chains = synth.generate_corpus(p, 0)
dc = fg.DeviceCorpus(c)
ix = fg.build_hybrid_index(dc, kg, degree=16, knn_k=32, seed=5100)
for i, ch in enumerate(chains):
    q = A.Queries(ch.query_dense[None, :], A.CSR.from_rows([ch.query_learned[0]], [ch.query_learned[1]]),
                  A.CSR.from_rows([ch.query_statistical[0]], [ch.query_statistical[1]]),
                  np.array([[1, 1, 1, 100]], np.float32), k=10, beam_width=128, max_entity_hops=2,
                  entities=A.CSR.from_rows([[ch.e0]]))
    r = fg.batch_query(ix, q)
    print(i, r.hit_count[0], r.expanded[0], flush=True)
