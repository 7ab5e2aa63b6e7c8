"""Profiling driver for the build: NN-Descent init + passes + refine on a
C2-shaped corpus, with per-pass wall times (run under ncu with
-k regex:knn_pass -c 1 to capture pass 1)."""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_00855_b200 import _abi as A, fusegraph as fg, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--docs", type=int, default=200000)
ap.add_argument("--k", type=int, default=64)
ap.add_argument("--passes", type=int, default=10)
a = ap.parse_args()
p = A.synth_params(docs=a.docs, dense_dim=768, learned_vocab=30522, learned_nnz=120,
                   statistical_vocab=0, statistical_nnz=40, seed=1)
c, kg, _ = synth.generate_corpus(p, 0)
dc = fg.DeviceCorpus(c)
t = time.time()
lists = fg.init_random_graph(dc, a.k, 42)
print(f"init {time.time() - t:.2f}s", flush=True)
for i in range(a.passes):
    t = time.time()
    *lists, changed = fg.nn_descent_iterate(dc, *lists)
    print(f"pass {i + 1}: {time.time() - t:.2f}s changed {changed} ({changed / (c.n * a.k):.4f})",
          flush=True)
    if changed / (c.n * a.k) < 0.01:
        break
t = time.time()
fg.refine_graph(dc, *lists, degree=32)
print(f"refine {time.time() - t:.2f}s", flush=True)
