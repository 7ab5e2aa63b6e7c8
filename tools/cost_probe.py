"""Dev probe: per-query work (scored nodes, expansions) of the bench's timed
batch against its fusion weight alpha — is the batch's tail a cost-variance
effect (longest-first dispatch could help) or granularity?

  python tools/cost_probe.py [--docs 1000000]"""
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
a = ap.parse_args()
p = bench.synth_params(a.docs)
c, kg, _ = synth.generate_corpus(p, 0)
ix = fg.build_hybrid_index(fg.DeviceCorpus(c), kg, **bench.BUILD)
op = bench.OPERATING_POINT
q = bench.c2_queries(p, a.queries, bench.TIMED_STREAM).with_(beam_width=op["beam"])
r = fg.batch_query(ix, q, entry_count=op["entry"])
alpha = q.weights[:, 0].astype(np.float64)
sc = r.scored.astype(np.float64)
ex = r.expanded.astype(np.float64)
print(f"scored mean {sc.mean():.0f} cv {sc.std() / sc.mean():.3f} p10 {np.percentile(sc, 10):.0f} "
      f"p90 {np.percentile(sc, 90):.0f} max {sc.max():.0f}; expanded mean {ex.mean():.1f} cv {ex.std() / ex.mean():.3f}")
print(f"corr(scored, alpha) {np.corrcoef(sc, alpha)[0, 1]:.3f}")
for lo in np.arange(0, 1, 0.1):
    m = (alpha >= lo) & (alpha < lo + 0.1)
    print(f"  alpha [{lo:.1f},{lo + 0.1:.1f}): n {m.sum():5d} scored {sc[m].mean():7.0f} expanded {ex[m].mean():6.1f}")
np.savez(os.path.join(ROOT, "gpurun_out", "cost_probe.npz"), alpha=alpha, scored=sc, expanded=ex)
