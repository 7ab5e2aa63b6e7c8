import os, sys, time
sys.path.insert(0, os.getcwd())
import bench
from paper_2511_00855_b200 import fusegraph as fg, synth
p = bench.synth_params(1_000_000)
c, kg, _ = synth.generate_corpus(p, 0)
for i in range(2):
    t0 = time.time(); dc = fg.DeviceCorpus(c); print("upload", time.time() - t0, flush=True); dc.close()
