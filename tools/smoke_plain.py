import sys, numpy as np
sys.path.insert(0, '/root/repo')
from paper_2511_00855_b200 import _abi as A, fusegraph as fg, synth
p = A.synth_params(docs=600, dense_dim=64, learned_vocab=2000, learned_nnz=24, statistical_vocab=2000, statistical_nnz=12, seed=11)
c, kg, _ = synth.generate_corpus(p, 0)
dc = fg.DeviceCorpus(c)
ix = fg.build_hybrid_index(dc, kg, degree=8, knn_k=16, seed=42)
q = synth.synth_queries(p, 8, beam_width=40)
r = fg.batch_query(ix, q, entry_count=48)
print("ok", r.hit_count[:4], r.expanded[:4])
