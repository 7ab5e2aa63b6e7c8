"""Builds the C2-shaped index once and prints stage times plus a digest of the
graph (dev: compare build variants / env settings, e.g. FGB_KNN_TIMING=1)."""
import argparse
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_00855_b200 import _abi as A, fusegraph as fg, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--docs", type=int, default=1000000)
ap.add_argument("--repeat", type=int, default=1, help="build this many times in one process")
ap.add_argument("--shape", default="C2", choices=["C2", "C3"], help="C3: + statistical vocab 831,592, nnz 40")
a = ap.parse_args()
p = A.synth_params(docs=a.docs, dense_dim=768, clusters=20, cluster_spread=0.25, learned_vocab=30522, learned_nnz=120,
                   statistical_vocab=831592 if a.shape == "C3" else 0, statistical_nnz=40, seed=1)
c, kg, _ = synth.generate_corpus(p, 0)
dc = fg.DeviceCorpus(c)
import time  # noqa: E402
for rep in range(a.repeat):
    t_wall = time.time()
    ix = fg.build_hybrid_index(dc, kg, degree=32, knn_k=64, knn_iterations=10, seed=42)
    t_wall = time.time() - t_wall
    g = ix.export()
    h = hashlib.md5(g["semantic"].tobytes() + g["norm_order"].tobytes()).hexdigest()[:12]
    t = {k: round(float(v), 3) for k, v in ix.build_times().items()}
    print(f"env {' '.join(f'{k}={v}' for k, v in os.environ.items() if k.startswith('FGB_'))} build {t} "
          f"wall {t_wall:.2f}s graph {h}", flush=True)
    ix.close()
