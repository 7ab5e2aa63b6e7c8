"""Dev probe: A/B one environment knob on plain batches of a config shape,
alternating settings inside one process (box-to-box variance is ~10%).

  python tools/ab_env.py --config C4 --env FGB_SEARCH_CUCKOO --values 0,1 [--queries 10000]"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2511_00855_b200 import _abi as A, fusegraph as fg, synth  # noqa: E402
from tools.config_bench import CONFIGS  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C4")
    ap.add_argument("--docs", type=int, default=200000)
    ap.add_argument("--queries", type=int, default=10000)
    ap.add_argument("--beam", type=int, default=672)
    ap.add_argument("--entry", type=int, default=256)
    ap.add_argument("--env", required=True)
    ap.add_argument("--values", default="0,1")
    ap.add_argument("--rounds", type=int, default=3)
    a = ap.parse_args()
    cfg = dict(CONFIGS[a.config])
    cfg.pop("queries", None)
    cfg["docs"] = a.docs
    if "chains" in cfg:
        cfg["chains"] = min(cfg["chains"], a.docs // 1000)
    p = A.synth_params(**cfg)
    c, kg, _ = synth.generate_corpus(p, 0)
    ix = fg.build_hybrid_index(fg.DeviceCorpus(c), kg, **bench.BUILD)
    q = synth.synth_queries(p, a.queries, beam_width=a.beam)
    vals = a.values.split(",")
    best = {v: float("inf") for v in vals}
    res = {}
    for _ in range(a.rounds):
        for v in vals:
            os.environ[a.env] = v
            bench.flush_l2(0)
            r = fg.batch_query(ix, q, entry_count=a.entry)
            best[v] = min(best[v], ix.last_search_stats()[0])
            res[v] = r
    key = [(res[v].node, res[v].score, res[v].hit_count, res[v].expanded) for v in vals]
    same = all(all(np.array_equal(x, y) for x, y in zip(key[0], k)) for k in key[1:])
    for v in vals:
        print(f"{a.env}={v:6s} {ix.last_search_kernel():22s} {a.queries / (best[v] / 1e3):10.1f} QPS "
              f"({best[v]:.2f} ms)", flush=True)
    print("identical results:", same)


if __name__ == "__main__":
    main()
