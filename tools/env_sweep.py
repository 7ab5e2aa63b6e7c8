"""Builds (or loads) one C2-shaped index, then times batch_query under several
environment settings read per call by the library (FGB_SEARCH_*), e.g.
  python tools/env_sweep.py --docs 1000000 --set FGB_SEARCH_PREFETCH=1 --set FGB_SEARCH_PREFETCH=5
Each --set is 'K=V[,K2=V2]'; 'timing' adds FGB_SEARCH_TIMING=1 for one extra call."""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_00855_b200 import _abi as A, fusegraph as fg, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--docs", type=int, default=1000000)
ap.add_argument("--queries", type=int, default=10000)
ap.add_argument("--beam", type=int, default=512)
ap.add_argument("--entry", type=int, default=256)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--set", action="append", default=[])
ap.add_argument("--timing", action="store_true")
a = ap.parse_args()
p = A.synth_params(docs=a.docs, dense_dim=768, learned_vocab=30522, learned_nnz=120,
                   statistical_vocab=0, statistical_nnz=40, seed=1)
c, kg, _ = synth.generate_corpus(p, 0)
dc = fg.DeviceCorpus(c)
cache = f"/tmp/fgb_sweep_graph_{a.docs}.npz"  # reused by later commands of the same gpurun call
if os.path.exists(cache):
    z = np.load(cache)
    g = dict(degree=int(z["degree"]), semantic=z["semantic"], keyword=A.CSR(z["kp"], z["ki"]),
             logical_ptr=z["lp"], logical=z["lg"], norm_order=z["no"])
    ix = fg.HybridIndex.from_graph(dc, g, kg)
else:
    ix = fg.build_hybrid_index(dc, kg, degree=32, knn_k=64, knn_iterations=10, seed=42)
    print("build", ix.build_times(), flush=True)
    g = ix.export()
    np.savez(cache, degree=g["degree"], semantic=g["semantic"], kp=g["keyword"].ptr, ki=g["keyword"].idx,
             lp=g["logical_ptr"], lg=g["logical"], no=g["norm_order"])
print("library", os.environ.get("FGB_LIB_VARIANT", "default"), flush=True)
q = synth.synth_queries(p, a.queries).with_(beam_width=a.beam)
ref = None
for spec in a.set or [""]:
    kv = dict(x.split("=", 1) for x in spec.split(",") if x)
    old = {k: os.environ.get(k) for k in kv}
    os.environ.update(kv)
    best = 0.0
    for _ in range(a.reps):
        r = fg.batch_query(ix, q, entry_count=a.entry)
        ms, _ = ix.last_search_stats()
        best = max(best, q.count / (ms / 1e3))
    if ref is None:
        ref = r
    same = np.array_equal(ref.node, r.node) and np.array_equal(ref.score.view(np.uint64), r.score.view(np.uint64))
    import hashlib
    h = hashlib.md5(r.node.tobytes() + r.score.tobytes() + r.expanded.tobytes()).hexdigest()[:12]
    print(f"{spec or 'default'}: {best:.0f} QPS kernel (best of {a.reps}), scored {r.scored.mean():.0f}, "
          f"expanded {r.expanded.mean():.1f}, identical {same}, results {h}", flush=True)
    if a.timing:
        os.environ["FGB_SEARCH_TIMING"] = "1"
        fg.batch_query(ix, q, entry_count=a.entry)
        del os.environ["FGB_SEARCH_TIMING"]
    for k, v in old.items():
        if v is None:
            os.environ.pop(k, None)
        else:
            os.environ[k] = v
