"""Regenerate tests/golden/*.npz from the UNMODIFIED reference (oracle/_ref).

  python tests/golden/make_golden.py

Inputs come from the reference's own generate_corpus / random_query_vector /
random_simplex_weights (via the glue), so the fixtures pin the whole path:
corpus bytes, squared norms, hybrid scores, NN-Descent (init, one pass, full
build), the refinery trace, the built index, batched search (plain, keyword
and entity queries, error rows) and exhaustive truth.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from paper_2511_00855_b200 import _abi as A  # noqa: E402
from oracle.refpy import RefLib  # noqa: E402

PARAMS = dict(docs=600, dense_dim=16, learned_vocab=1200, learned_nnz=12, statistical_vocab=1200,
              statistical_nnz=10, entity_vocab=120, kg_triplets=400, chains=6,
              answers_per_chain=3, seed=21)
BUILD = dict(degree=6, knn_k=12, knn_iterations=10, seed=5, logical_cap=8)


def queries(ref, p, n=24, beam=20):
    d, li, lv, si, sv, w = ref.synth_queries(p, n)
    ln = len(li) // n
    sn = len(si) // n
    q = A.Queries(d, A.CSR(np.arange(n + 1) * ln, li, lv), A.CSR(np.arange(n + 1) * sn, si, sv), w,
                  k=8, beam_width=beam)
    rows = [q.statistical.row(i)[0][: i % 3].tolist() if i % 4 == 0 else [] for i in range(n)]
    q.required = A.CSR.from_rows(rows)
    q.k[5] = 0  # invalid-k row
    return q


def results_dict(prefix, r):
    return {f"{prefix}_count": r.hit_count, f"{prefix}_doc": r.doc_id, f"{prefix}_score": r.score,
            f"{prefix}_expanded": r.expanded, f"{prefix}_warn": r.warnings,
            f"{prefix}_err": np.array([r.error(i) for i in range(r.count)])}


def main():
    ref = RefLib()
    p = A.synth_params(**PARAMS)
    c, kg, nch = ref.generate_corpus(p)
    st = ref.store(c, kg)
    out = dict(dense=c.dense, lptr=c.learned.ptr, lidx=c.learned.idx, lval=c.learned.val,
               sptr=c.statistical.ptr, sidx=c.statistical.idx, sval=c.statistical.val,
               eptr=c.entities.ptr, eidx=c.entities.idx, kg_s=kg.source, kg_r=kg.relation,
               kg_t=kg.target, sqnorm=ref.sqnorm(st, c.n))
    q = queries(ref, p)
    ids = np.arange(c.n, dtype=np.uint32)
    out["scores_q0"] = ref.batch_scores(st, q, 0, ids)
    out["scores_q1"] = ref.batch_scores(st, q, 1, ids)
    i0 = ref.knn_init(st, c.n, BUILD["knn_k"], BUILD["seed"])
    i1 = ref.knn_iterate(st, *i0)
    kb = ref.knn_build(st, c.n, BUILD["knn_k"], max_iterations=10, seed=BUILD["seed"])
    out.update(init_ids=i0[0], init_sc=i0[1], pass_ids=i1[0], pass_sc=i1[1], pass_fr=i1[2],
               pass_changed=np.array(i1[3]), knn_ids=kb[0], knn_sc=kb[1], knn_fr=kb[2])
    sem, kw, tr = ref.refine(st, *kb, degree=BUILD["degree"], trace=True)
    out.update(ref_sem=sem, ref_kwc=np.array([len(x) for x in kw]),
               ref_kw=np.concatenate(kw) if kw else np.zeros(0, np.uint32),
               ref_ord=tr["ordered_ids"], ref_det=tr["detours"], ref_keptc=tr["kept_count"])
    ix = ref.index_build(ref.store(c, kg), **BUILD)
    g = ref.index_export(ix, c.n)
    out.update(ix_sem=g["semantic"], ix_kptr=g["keyword"].ptr, ix_kidx=g["keyword"].idx,
               ix_lptr=g["logical_ptr"], ix_lg=g["logical"], ix_norm=g["norm_order"])
    out.update(results_dict("plain", ref.batch_query(ix, q)))
    # entity queries from the planted chains: weights (1,1,1,100)
    qt = q.with_(k=8)  # brute_force_topk throws on invalid k; use a valid batch
    out.update(results_dict("truth", ref.brute_force(ref.store(c, kg), qt)))
    np.savez_compressed(os.path.join(HERE, "golden_small.npz"), **out)
    print("wrote", os.path.join(HERE, "golden_small.npz"))


if __name__ == "__main__":
    main()
