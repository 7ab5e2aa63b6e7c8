"""The refinery's tensor-core candidate Gram (refine.cu gram_tc_*): the dense
half of candidate_pair_scores (refine.cpp:11-23) on tcgen05 as a certified
split-bf16 product, every pair within the error bound of a decision threshold
re-scored with the reference's exact fp64 chain.

Checks, against the UNMODIFIED reference (oracle/_ref), bit for bit:
  * the refine trace (ordered candidates, detours, kept lists) and the
    semantic/keyword edges, for M=64 (k <= 64) and M=128 (k <= 128) MMA
    shapes, d=768 and a dense dim that is not a multiple of the 64-wide K
    chunk (zero padding);
  * the same with the bound inflated x1e6 (every pair resolved exactly) and
    with the tensor cores off (FGB_REFINE_TC=0, the SIMT fp64 Gram);
and that the measured error of the tensor-core dense products stays a safe
factor (>= 3x) below the bound the certification assumes (2^-10 |x||y|).
"""
import os

import numpy as np
import pytest

from paper_2511_00855_b200 import _abi as A, fusegraph as fg, synth

pytestmark = pytest.mark.gpu
THREADS = os.cpu_count() or 1
TC_EPS = 2.0 ** -10


def _case(ref, docs, dense_dim, k, **kw):
    p = A.synth_params(docs=docs, dense_dim=dense_dim, clusters=20, cluster_spread=0.25, seed=17, **kw)
    c, kg, _ = synth.generate_corpus(p, 0)
    dev = fg.DeviceCorpus(c)
    st = ref.store(c, kg)
    lists = ref.knn_build(st, c.n, k, max_iterations=3, seed=42, threads=THREADS)
    return dev, st, lists


def _same_refine(ref, dev, st, lists, degree):
    gs, gk, gt = fg.refine_graph(dev, *lists, degree=degree, trace=True)
    rs, rk, rt = ref.refine(st, *lists, degree=degree, threads=THREADS, trace=True)
    for key in ("ordered_ids", "detours", "kept_count"):
        assert np.array_equal(gt[key], rt[key]), key
    kc = gt["kept_count"]
    mask = np.arange(gt["kept"].shape[1])[None, :] < kc[:, None]
    assert np.array_equal(np.where(mask, gt["kept"], 0), np.where(mask, rt["kept"], 0))
    assert np.array_equal(gs, rs)
    assert all(np.array_equal(a, b) for a, b in zip(gk, rk))


@pytest.mark.parametrize("dense_dim,k,degree", [(768, 64, 32), (70, 24, 8), (96, 100, 32), (768, 15, 8)])
def test_tc_gram_identical_and_within_bound(ref, monkeypatch, dense_dim, k, degree):
    dev, st, lists = _case(ref, 3000, dense_dim, k, learned_vocab=30522, learned_nnz=40,
                           statistical_vocab=5000, statistical_nnz=12)
    monkeypatch.setenv("FGB_REFINE_TC_CHECK", "1")
    fg.refine_tc_stats(reset=True)
    _same_refine(ref, dev, st, lists, degree)
    s = fg.refine_tc_stats(reset=True)
    assert s["pairs"] == 3000 * k * (k - 1) // 2, s          # the tensor-core path ran for every pair
    assert 0.0 < s["max_rel_err"] < TC_EPS / 3, s            # the bound holds with margin
    assert s["resolved"] < s["pairs"] // 10, s               # certification decides most pairs


def test_tc_gram_forced_resolution_and_simt_fallback(ref, monkeypatch):
    dev, st, lists = _case(ref, 2000, 768, 64, learned_vocab=30522, learned_nnz=60,
                           statistical_vocab=0, statistical_nnz=0)
    monkeypatch.setenv("FGB_REFINE_TC_STATS", "1")
    monkeypatch.setenv("FGB_REFINE_TC_EPS_SCALE", "1e6")      # every pair uncertain -> exact
    fg.refine_tc_stats(reset=True)
    _same_refine(ref, dev, st, lists, 32)
    s = fg.refine_tc_stats(reset=True)
    assert s["resolved"] == s["pairs"] > 0, s
    monkeypatch.delenv("FGB_REFINE_TC_EPS_SCALE")
    monkeypatch.setenv("FGB_REFINE_TC", "0")                 # exact SIMT fp64 Gram
    _same_refine(ref, dev, st, lists, 32)
    assert fg.refine_tc_stats(reset=True)["pairs"] == 0
