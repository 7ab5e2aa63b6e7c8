#!/usr/bin/env python
"""bench.py — hybrid-query QPS at recall@10 >= 0.9 and index build seconds
(BASELINE.json `metric`) on the configs[1] workload: 1M docs, MS MARCO-shaped
(dense d=768 + SPLADE-like learned sparse, vocab 30,522, nnz 120), dense+sparse
fusion with per-query weights (alpha, 1-alpha, 0, 0), alpha ~ U[0,1) per query
(SURVEY §8 C2), built with degree 32 / knn_k 64 / 10 passes / seed 42.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--sweep]

One step = one batched beam search of this rank's query shard (the index is
replicated per GPU; queries shard by contiguous range, no collective on the
data path -> "scaling": "weak" in queries per GPU).

Operating point.  The (SearchOptions::entry_count, beam_width) pair — both
query-time options of the reference API, with identical results on both arms
— is the committed OPERATING_POINT below, selected by `--sweep` on a HELD-OUT
query set (stream 0x71E6, disjoint from the timed batch, stream 0x71E5): the
fastest setting whose mean recall@10 against exact truth reaches 0.9 with a
0.005 margin (profiles/r02_sweep.json).  Every run then measures recall@10 on
the first --eval-queries of the TIMED batch against exact GPU brute-force truth
(`brute_force_topk`, itself bit-identical to the reference's eval.cpp:14-51).
The reference arm uses the same constant, so both arms time the same config.

`value` = queries / device time of the search kernel (CUDA events on the
library's stream, max over ranks); `e2e` = queries / wall time of the public
C-ABI call with host buffers (H2D of the queries + D2H of the hits inside).
L2 is flushed (256 MiB write) before every timed step; the corpus (4 GB) is
larger than L2 as well.  `build_seconds` = host->device corpus upload and
packing + build_hybrid_index (max over ranks).

In-run CPU references (rank 0, N=1; oracle/_ref = the UNMODIFIED reference
compiled from /root/reference, loaded only as the checker/baseline):
  cpu_baseline        fusegraph_ref::batch_query over the same 1M index (loaded
                      from the GPU build's HYBGRIX1 bytes), all host threads,
                      on the first --cpu-sample queries of the timed batch;
                      plus a 1-thread row and the lscpu model
  parity_1m           those queries' GPU hits vs the reference's hits: ids,
                      score bits, hit counts and `expanded`, all identical
  build_cpu_baseline  fusegraph_ref::build_hybrid_index at configs[0] (10K
                      docs) on all host threads vs the GPU build of the same
                      corpus (upload included), semantic edges compared

--impl reference times the UNMODIFIED reference's batch_query (oracle/_ref,
all host threads) over the same index on --cpu-sample queries per step.  The
index fixture is built by a separate process (`bench.py --make-fixture`: GPU
build -> HYBGRIX1 file, the reference's own on-disk format) and loaded with
fusegraph_ref::deserialize_index, so the timing process never maps the B200
library (a CPU build at 1M takes hours).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "hybrid-query QPS at recall@10>=0.9 (1/2/4/8 B200) and index build seconds"
BEAMS = [16, 32, 64, 128, 256, 512, 1024, 2048]
# SearchOptions::entry_count (search.hpp:45-49): the number of largest-norm
# entry points (index.cpp:15-22).
ENTRIES = [32, 64, 128, 256, 512, 1024]
# selected by `python bench.py --sweep` on the held-out stream (profiles/r02_sweep.json)
OPERATING_POINT = {"entry": 512, "beam": 480}
TIMED_STREAM, HELDOUT_STREAM = 0x71E5, 0x71E6
WORKLOAD = ("configs[1]: 1M docs MS MARCO-shaped dense d=768 + learned sparse nnz 120 "
            "(vocab 30522), dense+sparse fusion, per-query weights (a, 1-a, 0, 0), a~U[0,1)")
# configs[4] (C5): 10M docs shaped as configs[1], 100K-query batches sharded
# over the GPUs, build sharded by vertex range.  Operating point: entry 256
# (round 1's sweep); beam 3008 gave recall 0.9005 on round 1's sample and
# 0.8995 on the timed batch (round 2), so the default is 10% above it.
C5 = dict(docs=10_000_000, queries=100_000, point={"entry": 256, "beam": 3328},
          workload=("configs[4]: 10M docs shaped as configs[1] (dense d=768 + learned sparse nnz 120), "
                    "100K-query batches sharded over the GPUs, index replicated, build sharded by vertex range"))

BUILD = dict(degree=32, knn_k=64, knn_iterations=10, seed=42, logical_cap=64)
C1 = dict(docs=10000, dense_dim=128, clusters=20, cluster_spread=0.25, learned_vocab=30000,
          learned_nnz=64, statistical_vocab=30000, statistical_nnz=64, seed=1)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--docs", type=int, default=1_000_000)
    ap.add_argument("--queries", type=int, default=10_000)
    ap.add_argument("--eval-queries", type=int, default=1000)
    ap.add_argument("--cpu-sample", type=int, default=1024)
    ap.add_argument("--beam", type=int, default=0, help="override the operating point's beam")
    ap.add_argument("--entry", type=int, default=0, help="override the operating point's entry_count")
    ap.add_argument("--sweep", action="store_true",
                    help="re-select the operating point on the held-out stream (printed in the line)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-build-baseline", action="store_true")
    ap.add_argument("--make-fixture", default="", help=argparse.SUPPRESS)
    ap.add_argument("--config", default="C2", choices=["C2", "C5"],
                    help="C2 = configs[1] (the driver's default); C5 = configs[4] at 10M docs")
    a = ap.parse_args()
    if a.config == "C5":
        if a.docs == 1_000_000:
            a.docs = C5["docs"]
        if a.queries == 10_000:
            a.queries = C5["queries"]
    return a


def synth_params(docs):
    from paper_2511_00855_b200 import _abi as A
    return A.synth_params(docs=docs, dense_dim=768, clusters=20, cluster_spread=0.25,
                          learned_vocab=30522, learned_nnz=120, statistical_vocab=0,
                          statistical_nnz=40, seed=1)


def c2_weights(count, stream):
    """(alpha, 1-alpha, 0, 0), alpha ~ U[0,1) in fp32 per query."""
    a = np.random.default_rng(stream).random(count).astype(np.float32)
    w = np.zeros((count, 4), np.float32)
    w[:, 0] = a
    w[:, 1] = np.float32(1.0) - a
    return w


def c2_queries(p, count, stream, gen=None):
    """Query vectors from the reference generator's stream (random_query_vector,
    fusegraph_cli.cpp:184-194) with C2's two-path weights.  `gen` = a RefLib
    (reference arm: no B200 library in that process) or None (synth.py)."""
    from paper_2511_00855_b200 import _abi as A
    if gen is None:
        from paper_2511_00855_b200 import synth
        q = synth.synth_queries(p, count, stream=stream)
    else:
        dense, li, lv, si, sv, _ = gen.synth_queries(p, count, stream=stream)
        ln = min(p.learned_nnz, p.learned_vocab)
        sn = min(p.statistical_nnz, p.statistical_vocab)
        lp = np.arange(count + 1, dtype=np.uint64) * np.uint64(ln)
        sp = np.arange(count + 1, dtype=np.uint64) * np.uint64(sn)
        q = A.Queries(dense, A.CSR(lp, li, lv), A.CSR(sp, si, sv), np.zeros((count, 4), np.float32))
    q.weights = c2_weights(count, stream)
    return q


class Clocks:
    """nvidia-smi sampler running during the timed region."""

    def __init__(self, device):
        self.path = f"/tmp/fgb_clocks_{os.getpid()}.csv"
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(device), f"--query-gpu={q}",
                                       "--format=csv,noheader,nounits", "-lms", "250"],
                                      stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if not self.p:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for nm, v in zip(names, f[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        os.unlink(self.path)
        busy = [s for s in sm if s > 0.5 * max(sm)] if sm else []
        return {"sm_mhz": statistics.median(busy) if busy else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


def peak_hbm():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def peak_bf16():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["bf16_tflops"]), "measured"
    except Exception:
        return 1590.0, "fallback"


def build_rooflines(fg, ix, corpus, stages):
    """Rooflines of the two construction kernels from this build's own
    counters: NN-Descent (algorithmic bytes = pair scores x row bytes, SURVEY
    8(d); the bytes the certified screening actually gathers beside it) and
    the refinery's tensor-core Gram (useful dense FLOPs = pairs x 2d)."""
    bs = ix.build_stats()
    R = row_bytes(corpus)
    peak, kind = peak_hbm()
    out = {}
    if bs["pass_seconds"] > 0:
        nl = corpus.learned.ptr[-1] / corpus.n
        ns = corpus.statistical.ptr[-1] / corpus.n
        # postings of every candidate the pass-1 sketches did not reject, the
        # 512-byte sketch of every sketched candidate, the dense rows read
        gathered = ((bs["candidates"] - bs["sketch_rejected"]) * 8 * (nl + ns) + bs["sketched"] * 512
                    + bs["dense_rows"] * 4 * corpus.dense_dim)
        alg = bs["candidates"] * R
        out["knn"] = {
            "bound": "hbm", "kernel": "knn_pass_kernel", "passes": bs["passes"], "pair_scores": bs["candidates"],
            "dense_rows_read": bs["dense_rows"], "device_seconds": round(bs["pass_seconds"], 3),
            "sketched": bs["sketched"], "sketch_rejected": bs["sketch_rejected"],
            "alg_bytes": int(alg), "achieved": round(alg / bs["pass_seconds"] / 1e9, 1), "peak": peak,
            "peak_kind": kind, "unit": "GB/s", "frac": round(alg / bs["pass_seconds"] / 1e9 / peak, 4),
            "gathered_bytes": int(gathered),
            "gathered_frac": round(gathered / bs["pass_seconds"] / 1e9 / peak, 4),
            "traffic_note": "pass 1 at 200K docs under ncu (sketch screening): 1.55 TB DRAM in 0.72 s = 0.33 "
                            "of peak (profiles/r02_knn_sketch_ncu.md)",
            "note": "alg_bytes counts every scored pair at full row bytes; the certified screening reads the "
                    "dense row of only dense_rows_read of them"}
    tc = fg.refine_tc_stats(reset=True)
    if tc["pairs"]:
        flops = tc["pairs"] * 2.0 * corpus.dense_dim
        tpk, tkind = peak_bf16()
        out["refine_gram"] = {
            "bound": "tensor", "kernel": "refine_node_kernel (tcgen05 split-bf16 Gram)", "pairs": tc["pairs"],
            "exact_rescored": tc["resolved"], "useful_dense_tflop": round(flops / 1e12, 3),
            "refine_seconds": round(stages.get("refine", 0.0), 3),
            "achieved": round(flops / max(stages.get("refine", 1e-9), 1e-9) / 1e12, 2), "peak": tpk,
            "peak_kind": tkind, "unit": "TFLOP/s",
            "frac": round(flops / max(stages.get("refine", 1e-9), 1e-9) / 1e12 / tpk, 5),
            "note": "one 64x64x768 Gram per node (x3 MMAs for the hi/lo split): the refine stage is bound by "
                    "the sparse merge-joins, not the tensor pipe (profiles/r02_refine_tc.md)"}
    return out


def cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def dist_setup(args):
    from paper_2511_00855_b200.shard import env_world
    world, rank, local = env_world()
    if world > 1 and args.impl != "reference":
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(device_of(local))
        if dist_backend() == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(dist_backend())
    return world, rank, local


def flush_l2(local):
    import torch
    buf = getattr(flush_l2, "buf", None)
    if buf is None:
        buf = flush_l2.buf = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{local}")
    buf.zero_()
    torch.cuda.synchronize(local)


def row_bytes(c):
    """Algorithmic bytes of one scored document."""
    nl = (c.learned.ptr[-1] / c.n) if c.n else 0
    ns = (c.statistical.ptr[-1] / c.n) if c.n else 0
    return 4 * c.dense_dim + 8 * nl + 8 * ns


def operating_point(args):
    pt = C5["point"] if getattr(args, "config", "C2") == "C5" else OPERATING_POINT
    return (args.entry or pt["entry"]), (args.beam or pt["beam"])


def dist_backend():
    """NCCL between GPUs; FGB_DIST_BACKEND=gloo runs several ranks on fewer
    GPUs (multi-rank tests on a one-GPU box: ranks share device rank % GPUs,
    the sharded build exchanges through the host communicator)."""
    return os.environ.get("FGB_DIST_BACKEND", "nccl")


def device_of(local):
    import torch
    return local % max(1, torch.cuda.device_count())


def load_corpus(p, world, rank, group):
    """The synthetic corpus of this run.  With several ranks on one host,
    rank 0 generates it once into /dev/shm and the others map those arrays
    (a 10M-doc corpus is ~41 GB of host memory per copy); FGB_BENCH_SHARED=0
    makes every rank generate its own."""
    from paper_2511_00855_b200 import _abi as A, synth
    if world == 1 or os.environ.get("FGB_BENCH_SHARED", "1") == "0" or not os.path.isdir("/dev/shm"):
        corpus, kg, _ = synth.generate_corpus(p, 0)
        return corpus, kg, None
    d = f"/dev/shm/fgb_corpus_{os.getppid()}_{p.docs}_{p.seed}"
    names = ["dense", "lp", "li", "lv", "sp", "si", "sv", "kp", "ki", "ep", "ei", "doc_id", "ks", "kr", "kt"]
    if rank == 0:
        corpus, kg, _ = synth.generate_corpus(p, 0)
        os.makedirs(d, exist_ok=True)
        c = corpus
        kw = c.keywords if c.keywords is not None else A.CSR.empty(c.n, False)
        en = c.entities if c.entities is not None else A.CSR.empty(c.n, False)
        for nm, x in zip(names, [c.dense, c.learned.ptr, c.learned.idx, c.learned.val, c.statistical.ptr,
                                 c.statistical.idx, c.statistical.val, kw.ptr, kw.idx, en.ptr, en.idx, c.doc_id,
                                 kg.source, kg.relation, kg.target]):
            np.save(os.path.join(d, nm + ".npy"), np.asarray(x) if x is not None else np.zeros(0))
    group.barrier()
    if rank != 0:
        z = {nm: np.load(os.path.join(d, nm + ".npy"), mmap_mode="r") for nm in names}
        corpus = A.Corpus(z["dense"], A.CSR(z["lp"], z["li"], z["lv"]), A.CSR(z["sp"], z["si"], z["sv"]),
                          A.CSR(z["kp"], z["ki"]), A.CSR(z["ep"], z["ei"]), z["doc_id"], None,
                          p.learned_vocab, p.statistical_vocab)
        kg = A.KG(z["ks"], z["kr"], z["kt"])
    return corpus, kg, d


def traffic_for(docs, entry, beam):
    """ncu dram bytes per launch of search_plain_kernel at this exact operating
    point (profiles/r02_search_traffic.json, one `ncu --set full` capture of
    the same kernel build); None when the capture is for another point."""
    path = os.path.join(ROOT, "profiles", "r02_search_traffic.json")
    try:
        t = json.load(open(path))
    except Exception:
        return None, None
    if (t.get("docs"), t.get("entry"), t.get("beam")) != (docs, entry, beam):
        return None, None
    return t.get("dram_bytes_per_launch"), t.get("alg_bytes_per_launch")


def main():
    args = parse()
    if args.make_fixture:
        return make_fixture(args)
    world, rank, local = dist_setup(args)
    if args.impl == "reference":
        return reference_arm(args, world, rank, local)

    from paper_2511_00855_b200 import fusegraph as fg, synth
    import torch
    from paper_2511_00855_b200.shard import Group, build_comm, shard_range

    dev = device_of(local)
    torch.cuda.set_device(dev)
    group = Group(world, device=f"cuda:{dev}" if dist_backend() == "nccl" else "cpu")
    t0 = time.time()
    p = synth_params(args.docs)
    corpus, kg, shm_dir = load_corpus(p, world, rank, group)
    t_gen = time.time() - t0
    if world > 1 and dist_backend() != "nccl":
        comm = fg.HostComm(world, rank, dev)  # ranks sharing GPUs: host-staged exchange
    else:
        comm = build_comm(world, rank, dev)
    # ---- build: corpus upload + packing + build_hybrid_index (vertex-range
    # sharded over the ranks with NCCL all-gathers per pass)
    os.environ.setdefault("FGB_REFINE_TC_STATS", "1")  # counters for the build roofline (a few atomics)
    group.barrier()
    t0 = time.time()
    dc = fg.DeviceCorpus(corpus, device=dev)
    t_up = time.time() - t0
    if comm is not None:
        ix = fg.build_hybrid_index_sharded(dc, kg, comm=comm, **BUILD)
    else:
        ix = fg.build_hybrid_index(dc, kg, **BUILD)
    torch.cuda.synchronize(dev)
    build_s = group.max(time.time() - t0)
    stages = ix.build_times()
    stages["upload"] = t_up
    build_roof = build_rooflines(fg, ix, corpus, stages)

    queries = c2_queries(p, args.queries, TIMED_STREAM)
    entry, beam = operating_point(args)
    sweep = None
    if args.sweep and rank == 0:
        held = c2_queries(p, args.eval_queries, HELDOUT_STREAM)
        htruth = fg.brute_force_topk(dc, held)
        sweep = sweep_operating_points(fg, ix, held, htruth, args)
        best = select_operating_point(sweep)
        entry, beam = best["entry"], best["beam"]
    beam = int(group.bcast(beam))
    entry = int(group.bcast(entry))

    # ---- recall@10 on a sample of the TIMED batch (not the selection set)
    recall = None
    if rank == 0:
        ev = queries.subset(np.arange(min(args.eval_queries, queries.count))).with_(beam_width=max(beam, 10))
        truth = fg.brute_force_topk(dc, ev)
        r = fg.batch_query(ix, ev, entry_count=entry)
        recall = float(np.mean([fg.recall_at_k(r.ids(i), truth.ids(i), 10) for i in range(ev.count)]))

    # ---- this rank's shard
    lo, hi = shard_range(queries.count, world, rank)
    shard = queries.subset(np.arange(lo, hi)).with_(beam_width=max(beam, 10))
    shard = shard.pinned()  # e2e inputs come from page-locked host memory
    for _ in range(args.warmup):
        fg.batch_query(ix, shard, entry_count=entry)

    clocks = Clocks(dev)
    kern_ms, wall_s, scored, expanded, launches = [], [], 0, 0, 0
    res = None
    for _ in range(args.steps):
        flush_l2(dev)
        group.barrier()
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        res = fg.batch_query(ix, shard, entry_count=entry)  # H2D queries + kernel + D2H hits
        torch.cuda.synchronize(dev)
        wall_s.append(time.perf_counter() - t0)
        ms, nl = ix.last_search_stats()
        kern_ms.append(ms)
        launches += nl
        scored, expanded = int(res.scored.sum()), int(res.expanded.sum())
    clk = clocks.stop()
    group.barrier()
    k_tot = group.max(sum(kern_ms) / 1e3)
    w_tot = group.max(sum(wall_s))
    n_total = queries.count * args.steps
    value = n_total / k_tot
    e2e = n_total / w_tot

    # roofline of the search kernel: algorithmic bytes / kernel time
    R = row_bytes(corpus)
    deg = BUILD["degree"]
    qbytes = shard.h2d_bytes()
    alg_bytes = scored * R + expanded * 4 * deg + qbytes
    achieved = alg_bytes / (statistics.mean(kern_ms) / 1e3) / 1e9
    peak, peak_kind = peak_hbm()
    traffic, traffic_alg = traffic_for(corpus.n, entry, beam) if world == 1 else (None, None)

    line = {
        "metric": METRIC,
        "value": round(value, 1),
        "unit": "queries/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(k_tot / args.steps * 1e3, 3),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f32 storage / f64 accumulate",
        "data": "synthetic (reference generate_corpus, bit-identical), seed 1",
        "config": {
            "workload": C5["workload"] if args.config == "C5" else WORKLOAD,
            "docs": corpus.n, "queries_per_step": queries.count, "queries_per_gpu": hi - lo,
            "k": 10, "beam": beam, "entry_count": entry, "build": BUILD,
            "operating_point": "held-out selection (bench.py --sweep, stream 0x71E6)"
                               if not (args.beam or args.entry) else "forced by --beam/--entry",
            "parallelism": f"query-shard x{world}, index replicated; build vertex-range x{world} "
                           f"({'NCCL' if dist_backend() == 'nccl' or world == 1 else 'host-staged ' + dist_backend()} "
                           f"all-gather)" + ("" if world <= torch.cuda.device_count()
                                             else f"; {world} ranks share {torch.cuda.device_count()} GPU(s)"),
            "l2": "flushed (256 MiB write) before each timed step; corpus 4 GB > L2",
        },
        "recall_at_10": round(recall, 4) if recall is not None else None,
        "recall_sample": f"first {min(args.eval_queries, queries.count)} queries of the timed batch "
                         "vs exact GPU brute-force truth",
        "recall_target_met": (recall >= 0.9) if recall is not None else None,
        "build_seconds": round(build_s, 2),
        "build_stages_s": {k: round(v, 3) for k, v in stages.items()},
        "gen_seconds": round(t_gen, 2),
        "e2e": {"value": round(e2e, 1), "unit": "queries/s", "h2d_bytes_per_step": int(qbytes),
                "d2h_bytes_per_step": int(shard.count * (10 * 20 + 4 * 8))},
        "gpu_launches": int(launches),
        "roofline": {"bound": "hbm", "kernel": "search_plain_kernel", "achieved": round(achieved, 1),
                     "peak": peak, "peak_kind": peak_kind, "unit": "GB/s", "frac": round(achieved / peak, 4),
                     "traffic": traffic,
                     "traffic_source": "profiles/r02_search_traffic.json (ncu --set full, same point)"
                                       if traffic else None,
                     "alg_bytes_per_launch": int(alg_bytes),
                     "per_query": {"scored": scored / max(shard.count, 1),
                                   "expanded": expanded / max(shard.count, 1), "row_bytes": R}},
        "clocks": clk,
        "build_roofline": build_roof,
    }
    if sweep is not None:
        line["sweep"] = {"queries": args.eval_queries, "stream": HELDOUT_STREAM, "points": sweep}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cb, parity = cpu_baseline(ix, queries, res, beam, entry, args.cpu_sample)
        line["cpu_baseline"] = cb
        line["parity_1m"] = parity
    if rank == 0 and world == 1 and not args.no_build_baseline:
        ix.close()
        dc.close()
        line["build_cpu_baseline"] = build_baseline()
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        group.barrier()
        if rank == 0 and shm_dir:  # every rank has uploaded its copy long ago
            import shutil
            shutil.rmtree(shm_dir, ignore_errors=True)
        dist.destroy_process_group()


def sweep_operating_points(fg, ix, ev, truth, args):
    """recall@10 / kernel QPS over entry_count x beam on the held-out set; per
    entry_count the beam sweep stops at the first power-of-two beam reaching
    0.9 (larger beams only cost more), then bisects (steps of 16) below it."""
    rows = []

    def point(e, b):
        r = fg.batch_query(ix, ev.with_(beam_width=max(b, 10)), entry_count=e)
        rec = float(np.mean([fg.recall_at_k(r.ids(i), truth.ids(i), 10) for i in range(ev.count)]))
        ms, _ = ix.last_search_stats()
        rows.append({"entry": e, "beam": b, "recall": round(rec, 4),
                     "qps_kernel": round(ev.count / (ms / 1e3), 1)})
        return rec

    for e in ENTRIES:
        lo = 0
        for b in BEAMS:
            if point(e, b) >= 0.905:
                hi = b
                while hi - lo > 32:
                    mid = (lo + hi) // 32 * 16
                    if mid <= lo or mid >= hi:
                        break
                    if point(e, mid) >= 0.905:
                        hi = mid
                    else:
                        lo = mid
                break
            lo = b
    return rows


def select_operating_point(sweep):
    ok = [s for s in sweep if s["recall"] >= 0.905]
    if ok:
        return max(ok, key=lambda s: s["qps_kernel"])
    return max(sweep, key=lambda s: s["recall"])


def export_fixture(ix, path):
    """The GPU-built index in the reference's own file format (HYBGRIX1 v1,
    io.cpp:242-671): what `fusegraph_ref::deserialize_index` loads."""
    ix.serialize(path)
    return path


def cpu_baseline(ix, queries, gpu_res, beam, entry, sample):
    """The reference's own batch_query on host cores over the same index
    (deserialized from the GPU build's HYBGRIX1 bytes), plus the bitwise
    comparison of its hits with the GPU's for the same queries."""
    from oracle.refpy import RefLib, ref_available
    if not ref_available():
        return ({"value": None, "unit": "queries/s", "cores": 0, "kind": "reference",
                 "sample": "oracle/_ref not built"}, None)
    ref = RefLib()
    cores = os.cpu_count() or 1
    with tempfile.TemporaryDirectory(prefix="fgb_fixture_") as td:
        t0 = time.time()
        rix = ref.index_deserialize(export_fixture(ix, os.path.join(td, "c2.hyb")))
        prep_s = time.time() - t0
    m = min(sample, queries.count)
    q = queries.subset(np.arange(m)).with_(beam_width=max(beam, 10))
    pq = ref.prepare_queries(q)
    t0 = time.perf_counter()
    rr = ref.batch_query_prepared(rix, pq, 0, m, 10, entry_count=entry, threads=cores)
    dt = time.perf_counter() - t0
    m1 = min(64, m)
    t0 = time.perf_counter()
    ref.batch_query_prepared(rix, pq, 0, m1, 10, entry_count=entry, threads=1)
    dt1 = time.perf_counter() - t0
    # parity at 1M: the GPU's hits for the same queries (rows 0..m-1 of the
    # timed batch on rank 0) against the reference's
    g = gpu_res
    ident = (np.array_equal(g.hit_count[:m], rr.hit_count)
             and np.array_equal(g.doc_id[:m], rr.doc_id)
             and np.array_equal(g.score[:m].view(np.uint64), rr.score.view(np.uint64))
             and np.array_equal(g.expanded[:m], rr.expanded))
    mism = int(sum(1 for i in range(m) if not (
        np.array_equal(g.doc_id[i], rr.doc_id[i])
        and np.array_equal(g.score[i].view(np.uint64), rr.score[i].view(np.uint64)))))
    parity = {"queries": m, "identical": bool(ident), "mismatched_queries": mism,
              "compared": "hit ids, hit count, score bits, expanded",
              "reference": "fusegraph_ref::batch_query over deserialize_index(GPU build)"}
    cb = {"value": round(m / dt, 2), "unit": "queries/s", "cores": cores, "kind": "reference",
          "cpu_model": cpu_model(),
          "sample": f"first {m} queries of the timed batch at beam {beam}, entry_count {entry}, same "
                    f"{ix.corpus.n}-doc index (fusegraph_ref::batch_query, {cores} threads; "
                    f"HYBGRIX1 save+load {prep_s:.0f}s untimed)",
          "single_thread": {"value": round(m1 / dt1, 2), "unit": "queries/s", "cores": 1,
                            "sample": f"first {m1} queries, threads=1"}}
    return cb, parity


def build_baseline():
    """configs[0] (10K docs, d=128, nnz 64/64; degree 32, knn_k 64): the
    reference's build_hybrid_index on all host threads vs the GPU build of the
    same corpus (upload + build), edges compared."""
    from oracle.refpy import RefLib, ref_available
    from paper_2511_00855_b200 import _abi as A, fusegraph as fg, synth
    import torch
    if not ref_available():
        return {"unavailable": "oracle/_ref not built"}
    ref = RefLib()
    cores = os.cpu_count() or 1
    p = A.synth_params(**C1)
    c, kg, _ = synth.generate_corpus(p, 0)
    gpu_s = []
    for _ in range(3):  # the first run pays module load / allocations; min of the rest
        torch.cuda.synchronize()
        t0 = time.time()
        dc = fg.DeviceCorpus(c)
        gix = fg.build_hybrid_index(dc, kg, **BUILD)
        torch.cuda.synchronize()
        gpu_s.append(time.time() - t0)
        g = gix.export()
        gix.close()
        dc.close()
    st = ref.store(c, kg)
    t0 = time.time()
    rix = ref.index_build(st, threads=cores, **BUILD)
    cpu_s = time.time() - t0
    r = ref.index_export(rix, c.n)
    same = bool(np.array_equal(g["semantic"], r["semantic"])
                and np.array_equal(g["keyword"].idx, r["keyword"].idx)
                and np.array_equal(g["norm_order"], r["norm_order"]))
    return {"workload": "configs[0]: 10K docs, d=128, learned+statistical nnz 64, degree 32, knn_k 64",
            "gpu_seconds": round(min(gpu_s[1:]), 3), "gpu_seconds_runs": [round(x, 3) for x in gpu_s],
            "cpu_seconds": round(cpu_s, 2), "cores": cores, "cpu_model": cpu_model(),
            "kind": "reference", "speedup": round(cpu_s / min(gpu_s[1:]), 1), "identical_index": same}


def make_fixture(args):
    """(subprocess of the reference arm) GPU-build the 1M index, write HYBGRIX1."""
    from paper_2511_00855_b200 import fusegraph as fg, synth
    p = synth_params(args.docs)
    corpus, kg, _ = synth.generate_corpus(p, 0)
    dc = fg.DeviceCorpus(corpus)
    ix = fg.build_hybrid_index(dc, kg, **BUILD)
    export_fixture(ix, args.make_fixture)
    return 0


def reference_arm(args, world, rank, local):
    if rank != 0:
        return 0
    from oracle.refpy import RefLib, ref_available
    if not ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libfgref.so not built"}))
        return 0
    ref = RefLib()
    cores = os.cpu_count() or 1
    entry, beam = operating_point(args)
    p = synth_params(args.docs)
    with tempfile.TemporaryDirectory(prefix="fgb_fixture_") as td:
        path = os.path.join(td, "c2.hyb")
        t0 = time.time()
        subprocess.run([sys.executable, os.path.abspath(__file__), "--make-fixture", path,
                        "--docs", str(args.docs)], check=True)
        t_fix = time.time() - t0
        t0 = time.time()
        rix = ref.index_deserialize(path)
        t_load = time.time() - t0
    q = c2_queries(p, min(args.cpu_sample, args.queries), TIMED_STREAM, gen=ref).with_(
        beam_width=max(beam, 10))
    pq = ref.prepare_queries(q)
    for _ in range(args.warmup):
        ref.batch_query_prepared(rix, pq, 0, min(q.count, 4 * cores), 10, entry_count=entry, threads=cores)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        ref.batch_query_prepared(rix, pq, 0, q.count, 10, entry_count=entry, threads=cores)
        times.append(time.perf_counter() - t0)
    v = q.count * args.steps / sum(times)
    sample = (f"first {q.count} queries/step of the configs[1] timed batch at beam {beam}, entry_count "
              f"{entry}, fusegraph_ref::batch_query with {cores} threads over the same 1M index "
              f"(fixture: GPU build in a subprocess -> HYBGRIX1 -> fusegraph_ref::deserialize_index, "
              f"{t_fix:.0f}s + {t_load:.0f}s untimed)")
    print(json.dumps({
        "impl": "reference",
        "metric": METRIC,
        "value": round(v, 2), "unit": "queries/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(statistics.mean(times) * 1e3, 2),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32 storage / f64 accumulate", "data": "synthetic (reference generate_corpus), seed 1",
        "config": {"workload": WORKLOAD, "beam": beam, "entry_count": entry, "k": 10,
                   "docs": args.docs, "queries_per_step": q.count, "build": BUILD},
        "cpu_baseline": {"value": round(v, 2), "unit": "queries/s", "cores": cores,
                         "cpu_model": cpu_model(), "kind": "reference", "sample": sample},
        "e2e": {"value": round(v, 2), "unit": "queries/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main() or 0)
