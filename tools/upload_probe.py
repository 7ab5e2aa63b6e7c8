"""Dev probe: corpus upload time (DeviceCorpus of the configs[1] corpus),
alternating FGB_UPLOAD_LOCK settings inside one process.

  python tools/upload_probe.py [--docs 1000000] [--rounds 3]"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2511_00855_b200 import fusegraph as fg, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--docs", type=int, default=1_000_000)
ap.add_argument("--rounds", type=int, default=3)
a = ap.parse_args()
c, kg, _ = synth.generate_corpus(bench.synth_params(a.docs), 0)
fg.DeviceCorpus(c).close()  # warm-up (context, pools)
for r in range(a.rounds):
    for v in ("1", "0"):
        os.environ["FGB_UPLOAD_LOCK"] = v
        t = time.perf_counter()
        dc = fg.DeviceCorpus(c)
        dt = time.perf_counter() - t
        dc.close()
        print(f"FGB_UPLOAD_LOCK={v} upload {dt:.3f} s", flush=True)
