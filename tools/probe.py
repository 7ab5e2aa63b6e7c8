"""Dev probe: build + search timings on a C2-shaped corpus of --docs documents.

  python tools/probe.py --docs 100000 --queries 1000
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
    ap.add_argument("--docs", type=int, default=100000)
    ap.add_argument("--dim", type=int, default=768)
    ap.add_argument("--nnz", type=int, default=120)
    ap.add_argument("--vocab", type=int, default=30522)
    ap.add_argument("--stat-vocab", type=int, default=0)
    ap.add_argument("--stat-nnz", type=int, default=40)
    ap.add_argument("--queries", type=int, default=1000)
    ap.add_argument("--knn-k", type=int, default=64)
    ap.add_argument("--degree", type=int, default=32)
    ap.add_argument("--beams", default="16,32,64,128,256,512,1024")
    ap.add_argument("--eval", type=int, default=1000)
    a = ap.parse_args()
    out = {}
    p = A.synth_params(docs=a.docs, dense_dim=a.dim, learned_vocab=a.vocab, learned_nnz=a.nnz,
                       statistical_vocab=a.stat_vocab, statistical_nnz=a.stat_nnz, seed=1)
    t = time.time()
    c, kg, _ = synth.generate_corpus(p, 0)
    out["gen_s"] = time.time() - t
    t = time.time()
    dc = fg.DeviceCorpus(c)
    out["upload_s"] = time.time() - t
    cache = f"/tmp/fgb_graph_{a.docs}_{a.dim}_{a.nnz}_{a.knn_k}_{a.degree}.npz"
    t = time.time()
    if os.path.exists(cache):
        z = np.load(cache)
        g = dict(degree=int(z["degree"]), semantic=z["semantic"], keyword=A.CSR(z["kp"], z["ki"]),
                 logical_ptr=z["lp"], logical=z["lg"], norm_order=z["no"])
        ix = fg.HybridIndex.from_graph(dc, g, kg)
        out["build_s"] = "cached"
    else:
        ix = fg.build_hybrid_index(dc, kg, degree=a.degree, knn_k=a.knn_k, knn_iterations=10, seed=42)
        out["build_s"] = time.time() - t
        out["build_stages"] = ix.build_times()
        g = ix.export()
        np.savez(cache, degree=g["degree"], semantic=g["semantic"], kp=g["keyword"].ptr,
                 ki=g["keyword"].idx, lp=g["logical_ptr"], lg=g["logical"], no=g["norm_order"])
    q = synth.synth_queries(p, a.queries)
    t = time.time()
    truth = fg.brute_force_topk(dc, q.subset(np.arange(min(q.count, a.eval))))
    out["truth_s"] = time.time() - t
    rows = []
    for beam in [int(x) for x in a.beams.split(",")]:
        qb = q.with_(beam_width=max(beam, 10))
        t = time.time()
        r = fg.batch_query(ix, qb)
        wall = time.time() - t
        ms, _ = ix.last_search_stats()
        rec = np.mean([fg.recall_at_k(r.ids(i), truth.ids(i), 10) for i in range(truth.count)])
        rows.append(dict(beam=beam, recall=float(rec), qps_kernel=q.count / (ms / 1e3),
                         qps_wall=q.count / wall, scored=float(r.scored.mean()),
                         expanded=float(r.expanded.mean())))
        print(json.dumps(rows[-1]), flush=True)
    out["sweep"] = rows
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
