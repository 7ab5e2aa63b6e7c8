"""Dev probe: recall@10 vs beam / entry_count / build parameters on a
C2-shaped corpus (dense d=768 + learned nnz 120, simplex query weights).

  python tools/recall_probe.py --docs 200000 --builds 32:64,64:128 --beams 256,1024,4096
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_00855_b200 import _abi as A, fusegraph as fg, synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--docs", type=int, default=200000)
    ap.add_argument("--queries", type=int, default=500)
    ap.add_argument("--builds", default="32:64,64:128")
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--beams", default="256,512,1024,2048,4096")
    ap.add_argument("--entries", default="32")
    a = ap.parse_args()
    p = A.synth_params(docs=a.docs, dense_dim=768, clusters=20, cluster_spread=0.25,
                       learned_vocab=30522, learned_nnz=120, statistical_vocab=0,
                       statistical_nnz=40, seed=1)
    c, kg, _ = synth.generate_corpus(p, 0)
    dc = fg.DeviceCorpus(c)
    q = synth.synth_queries(p, a.queries)
    truth = fg.brute_force_topk(dc, q)
    for spec in a.builds.split(","):
        deg, k = (int(x) for x in spec.split(":"))
        t = time.time()
        ix = fg.build_hybrid_index(dc, kg, degree=deg, knn_k=k, knn_iterations=a.iters, seed=42)
        bs = time.time() - t
        print(json.dumps({"docs": a.docs, "degree": deg, "knn_k": k, "build_s": round(bs, 2),
                          "stages": {kk: round(v, 2) for kk, v in ix.build_times().items()}}), flush=True)
        for ec in (int(x) for x in a.entries.split(",")):
            for beam in (int(x) for x in a.beams.split(",")):
                r = fg.batch_query(ix, q.with_(beam_width=beam), entry_count=ec)
                ms, _ = ix.last_search_stats()
                rec = float(np.mean([fg.recall_at_k(r.ids(i), truth.ids(i), 10) for i in range(q.count)]))
                print(json.dumps({"degree": deg, "knn_k": k, "entry": ec, "beam": beam,
                                  "recall": round(rec, 4), "qps": round(q.count / (ms / 1e3), 1),
                                  "scored": float(r.scored.mean()),
                                  "expanded": float(r.expanded.mean())}), flush=True)
        ix.close()


if __name__ == "__main__":
    main()
