"""Dev probe: the plain search kernel's phase profile (FGB_SEARCH_TIMING=1)
and kernel QPS at the bench's configs[1] operating point, for A/B of search
kernel variants (FGB_LIB_VARIANT) and env knobs.

  python tools/search_phases.py [--docs 1000000] [--queries 10000]"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2511_00855_b200 import fusegraph as fg, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--docs", type=int, default=1_000_000)
ap.add_argument("--queries", type=int, default=10_000)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--no-timing", action="store_true")
ap.add_argument("--beam", type=int, default=0)
ap.add_argument("--entry", type=int, default=0)
a = ap.parse_args()
p = bench.synth_params(a.docs)
c, kg, _ = synth.generate_corpus(p, 0)
dc = fg.DeviceCorpus(c)
ix = fg.build_hybrid_index(dc, kg, **bench.BUILD)
entry = a.entry or bench.OPERATING_POINT["entry"]
beam = a.beam or bench.OPERATING_POINT["beam"]
q = bench.c2_queries(p, a.queries, bench.TIMED_STREAM).with_(beam_width=beam)
fg.batch_query(ix, q, entry_count=entry)
ms = []
for _ in range(a.reps):
    bench.flush_l2(0)
    fg.batch_query(ix, q, entry_count=entry)
    ms.append(ix.last_search_stats()[0])
print(f"{ix.last_search_kernel()} {q.count / (min(ms) / 1e3):.1f} QPS (best of {a.reps}: {min(ms):.2f} ms)", flush=True)
for pf in os.environ.get("ENV_SWEEP", "").split():  # NAME=VALUE settings, one measurement each
    name, val = pf.split("=")
    os.environ[name] = val
    ms = []
    for _ in range(a.reps):
        bench.flush_l2(0)
        fg.batch_query(ix, q, entry_count=entry)
        ms.append(ix.last_search_stats()[0])
    print(f"  {pf}: {q.count / (min(ms) / 1e3):.1f} QPS", flush=True)
    del os.environ[name]
if not a.no_timing:
    os.environ["FGB_SEARCH_TIMING"] = "1"
    fg.batch_query(ix, q, entry_count=entry)
