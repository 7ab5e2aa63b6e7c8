import sys, time, numpy as np
sys.path.insert(0, '/root/repo')
from paper_2511_00855_b200 import _abi as A, fusegraph as fg, synth
p = A.synth_params(docs=200000, dense_dim=768, learned_vocab=30522, learned_nnz=120, statistical_vocab=0, statistical_nnz=40, seed=1)
c, kg, _ = synth.generate_corpus(p, 0)
dc = fg.DeviceCorpus(c)
import os
cache = "/tmp/fgb_graph_200000_768_120_64_32.npz"
if os.path.exists(cache):
    z = np.load(cache)
    g = dict(degree=int(z["degree"]), semantic=z["semantic"], keyword=A.CSR(z["kp"], z["ki"]), logical_ptr=z["lp"], logical=z["lg"], norm_order=z["no"])
    ix = fg.HybridIndex.from_graph(dc, g, kg)
else:
    ix = fg.build_hybrid_index(dc, kg, degree=32, knn_k=64, seed=42)
q = synth.synth_queries(p, 10000).with_(beam_width=512)
for rep in range(4):
    t = time.perf_counter(); r = fg.batch_query(ix, q, entry_count=256); w = time.perf_counter() - t
    ms, _ = ix.last_search_stats()
    print(f"wall {w*1e3:.1f} ms kernel {ms:.1f} ms overhead {w*1e3-ms:.1f} ms")
