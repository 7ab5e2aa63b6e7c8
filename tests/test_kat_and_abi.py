"""Known-answer tests from the reference's own unit suites, run on the GPU
path and on the restatement oracle, plus the C-ABI contract checks (CPU)."""
import os
import re
import subprocess

import numpy as np
import pytest

from paper_2511_00855_b200 import _abi as A

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


# ----------------------------------------------------------------- C-ABI (CPU)
def test_library_exports_every_header_symbol():
    hdr = open(os.path.join(ROOT, "include", "fg_b200.h")).read()
    declared = set(re.findall(r"^\s*(?:int|const char\*)\s+(fg_\w+)\s*\(", hdr, re.M))
    assert len(declared) >= 25
    so = os.path.join(ROOT, "paper_2511_00855_b200", "libfgb200.so")
    out = subprocess.run(["nm", "-D", "--defined-only", so], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (fg_\w+)$", out, re.M))
    assert declared <= exported, declared - exported


def test_library_loads_and_reports_errors_without_gpu():
    from paper_2511_00855_b200 import Error, device_count, lib
    from paper_2511_00855_b200 import fusegraph as fg
    assert lib().fg_abi_version() == 1
    assert not lib().fgb_missing
    if device_count() == 0:  # no silent CPU fallback: compute must refuse
        c = A.Corpus(np.ones((3, 2), np.float32), A.CSR.empty(3), A.CSR.empty(3))
        with pytest.raises(Error) as e:
            fg.DeviceCorpus(c)
        assert e.value.code == "no-cuda-device"


def test_build_query_vector_host_matches_reference_rules():
    from paper_2511_00855_b200 import fusegraph as fg
    # corpus_test KAT (test_corpus.cpp:91-98): w=(0.5, 0, 2) -> dense halved,
    # learned dropped, statistical doubled
    q = A.Queries(np.array([[1.0, 2.0]], np.float32), A.CSR.from_rows([[3]], [[1.0]]),
                  A.CSR.from_rows([[5]], [[2.0]]), [[0.5, 0.0, 2.0, 0.0]])
    dense, lv, sv, sq = fg.build_query_vector(q, 0)
    assert dense.tolist() == [0.5, 1.0] and len(lv) == 0 and sv.tolist() == [4.0]
    assert sq == 0.25 + 1.0 + 16.0


# ----------------------------------------------------------------- KATs
def tiny(dense, learned=None, stat=None, entities=None):
    n = len(dense)
    return A.Corpus(np.asarray(dense, np.float32),
                    learned or A.CSR.empty(n), stat or A.CSR.empty(n), None,
                    entities or A.CSR.from_rows([[] for _ in range(n)]))


def dense_query(vec, w=(1, 0, 0, 0), k=2, beam=4, ents=None):
    q = A.Queries(np.array([vec], np.float32), A.CSR.empty(1), A.CSR.empty(1), [w], k=k,
                  beam_width=beam, entities=A.CSR.from_rows([ents or []]))
    return q


@pytest.mark.gpu
def test_kat_dense_and_sparse_hand_values():
    from paper_2511_00855_b200 import fusegraph as fg
    # test_scoring.cpp:68-71 / 86-93
    c = tiny([[0.5, 0.5], [3.0, 4.0]], learned=A.CSR.from_rows([[2, 7], [1, 4]], [[3.0, 1.0], [1.0, 1.0]]))
    dc = fg.DeviceCorpus(c)
    q = A.Queries(np.array([[1.0, 0.0], [3.0, 4.0]], np.float32),
                  A.CSR.from_rows([[2, 5], [2, 3]], [[1.0, 2.0], [1.0, 1.0]]), A.CSR.empty(2),
                  [[1, 1, 1, 0], [1, 1, 1, 0]])
    s0 = fg.batch_scores(dc, q, 0, [0])  # 0.5 + 3.0
    s1 = fg.batch_scores(dc, q, 1, [1])  # 25 + 0 (no shared terms)
    assert s0[0] == 3.5 and s1[0] == 25.0


@pytest.mark.gpu
def test_kat_three_node_exact_topk(oracle):
    from paper_2511_00855_b200 import fusegraph as fg
    # test_search.cpp:74-92: hits 0 (dot 1.0) then 1 (dot 0.8)
    c = tiny([[1.0, 0.0], [0.8, 0.5], [-1.0, 0.2]])
    dc = fg.DeviceCorpus(c)
    ix = fg.build_hybrid_index(dc, None, degree=2, knn_k=2, seed=42)
    r = fg.batch_query(ix, dense_query([1.0, 0.0]))
    assert r.hits(0)[0][0] == 0 and r.hits(0)[0][2] == 1.0
    assert r.hits(0)[1][0] == 1 and abs(r.hits(0)[1][2] - 0.8) < 1e-6


@pytest.mark.gpu
def test_kat_hop_reward_exactly_wk():
    from paper_2511_00855_b200 import fusegraph as fg
    # test_search.cpp:94-124: one logical hop earns exactly w_k / 1
    dense = [[2.0, 0.0], [0.0, 2.0]] + [[0.01 * i, 0.01] for i in range(2, 8)]
    ents = A.CSR.from_rows([[10], [11]] + [[] for _ in range(6)])
    c = tiny(dense, entities=ents)
    dc = fg.DeviceCorpus(c)
    ix = fg.build_hybrid_index(dc, A.KG([10], [0], [11]), degree=2, knn_k=4, seed=42)
    q = dense_query([1.0, 0.0], w=(1, 1, 1, 0.2), k=4, beam=8, ents=[10])
    r = fg.batch_query(ix, q)
    hits = {h[0]: h[2] for h in r.hits(0)}
    assert hits[0] == 2.0
    assert hits[1] == 0.0 + np.float64(np.float32(0.2))
