"""Refinery A/B: the tensor-core candidate Gram (default) vs the exact fp64
SIMT Gram (FGB_REFINE_TC=0) on a configs[1]-shaped corpus, plus the
certification counters (pairs, exact re-scores) and, on a node subset, the
measured max |tc - exact| / (|x||y|) against the 2^-10 bound.
  python tools/prof_refine_tc.py [--docs 200000] [--ncu]   (--ncu: one build, TC on)"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2511_00855_b200 import fusegraph as fg, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--docs", type=int, default=200_000)
ap.add_argument("--ncu", action="store_true")
a = ap.parse_args()
p = bench.synth_params(a.docs)
corpus, kg, _ = synth.generate_corpus(p, 0)
dc = fg.DeviceCorpus(corpus)
if a.ncu:
    fg.build_hybrid_index(dc, kg, **bench.BUILD)
    sys.exit(0)
out = {"docs": a.docs}
for mode in ("1", "0", "1"):
    os.environ["FGB_REFINE_TC"] = mode
    os.environ["FGB_REFINE_TC_STATS"] = mode
    fg.refine_tc_stats(reset=True)
    t0 = time.time()
    ix = fg.build_hybrid_index(dc, kg, **bench.BUILD)
    st = ix.build_times()
    key = "tc" if mode == "1" else "simt"
    out[key] = {"refine_s": round(st["refine"], 4), "knn_s": round(st["knn"], 3),
                "build_s": round(time.time() - t0, 3)}
    if mode == "1":
        s = fg.refine_tc_stats(reset=True)
        out[key].update(pairs=s["pairs"], resolved=s["resolved"],
                        resolved_frac=round(s["resolved"] / max(1, s["pairs"]), 6))
    g = ix.export()
    out.setdefault("semantic_equal", []).append(int(g["semantic"].sum()))
    ix.close()
out["semantic_equal"] = len(set(out["semantic_equal"])) == 1
# error calibration on a 20K-doc corpus of the same shape
p2 = bench.synth_params(20_000)
c2, kg2, _ = synth.generate_corpus(p2, 0)
d2 = fg.DeviceCorpus(c2)
os.environ["FGB_REFINE_TC"] = "1"
os.environ["FGB_REFINE_TC_CHECK"] = "1"
fg.refine_tc_stats(reset=True)
fg.build_hybrid_index(d2, kg2, **bench.BUILD)
s = fg.refine_tc_stats(reset=True)
out["calibration_20k"] = {"pairs": s["pairs"], "max_rel_err": s["max_rel_err"], "bound": 2.0 ** -10,
                          "margin": round(2.0 ** -10 / max(s["max_rel_err"], 1e-300), 2)}
print(json.dumps(out), flush=True)
