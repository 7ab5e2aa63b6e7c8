"""Profiling driver: one warm-up + one measured batched search on a C2-shaped
corpus (run under ncu with -k regex:search_kernel -s 1 -c 1)."""
import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_00855_b200 import _abi as A, fusegraph as fg, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--docs", type=int, default=100000)
ap.add_argument("--queries", type=int, default=2000)
ap.add_argument("--beam", type=int, default=256)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--entry", type=int, default=32)
ap.add_argument("--svocab", type=int, default=0, help="statistical vocabulary (C3: 831592)")
a = ap.parse_args()
p = A.synth_params(docs=a.docs, dense_dim=768, learned_vocab=30522, learned_nnz=120,
                   statistical_vocab=a.svocab, statistical_nnz=40, seed=1)
c, kg, _ = synth.generate_corpus(p, 0)
dc = fg.DeviceCorpus(c)
cache = f"/tmp/fgb_graph_{a.docs}_768_120_{a.svocab}_64_32.npz"
if os.path.exists(cache):
    z = np.load(cache)
    g = dict(degree=int(z["degree"]), semantic=z["semantic"], keyword=A.CSR(z["kp"], z["ki"]),
             logical_ptr=z["lp"], logical=z["lg"], norm_order=z["no"])
    ix = fg.HybridIndex.from_graph(dc, g, kg)
else:
    ix = fg.build_hybrid_index(dc, kg, degree=32, knn_k=64, knn_iterations=10, seed=42)
    g = ix.export()
    np.savez(cache, degree=g["degree"], semantic=g["semantic"], kp=g["keyword"].ptr,
             ki=g["keyword"].idx, lp=g["logical_ptr"], lg=g["logical"], no=g["norm_order"])
q = synth.synth_queries(p, a.queries).with_(beam_width=a.beam)
for _ in range(a.reps):
    t = time.time()
    r = fg.batch_query(ix, q, entry_count=a.entry)
    ms, _ = ix.last_search_stats()
    print(f"beam {a.beam}: {q.count / (ms / 1e3):.0f} QPS kernel, scored {r.scored.mean():.0f}, "
          f"expanded {r.expanded.mean():.0f}, wall {time.time() - t:.3f}s", flush=True)
