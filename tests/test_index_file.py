"""HYBGRIX1 v1 interop (io.cpp:242-671).

GPU: a GPU-built index serializes to exactly the bytes the UNMODIFIED
reference writes for its own (identical) build; the reference's
deserialize_index loads our file; a reference-written file loads into HBM and
searches bit-identically.  CPU: the reader's fault handling (checksum,
magic, version, truncation) uses the reference's error codes — the file is
rejected before anything touches a device (test_io.cpp:168-208)."""
import os
import struct

import numpy as np
import pytest

from paper_2511_00855_b200 import Error, _abi as A, fusegraph as fg, synth


@pytest.fixture(scope="module")
def ref_file(ref, tmp_path_factory):
    p = A.synth_params(docs=700, dense_dim=32, learned_vocab=2000, learned_nnz=16, statistical_vocab=2000,
                       statistical_nnz=12, entity_vocab=200, kg_triplets=600, chains=6, answers_per_chain=3,
                       seed=21)
    c, kg, _ = synth.generate_corpus(p, 0)
    rix = ref.index_build(ref.store(c, kg), degree=8, knn_k=16, seed=42, logical_cap=16)
    path = str(tmp_path_factory.mktemp("ix") / "ref.hybgrix")
    ref.index_serialize(rix, path)
    return p, c, kg, rix, path


def _load_err(path):
    with pytest.raises(Error) as e:
        fg.HybridIndex.deserialize(path)
    return e.value.code


def test_reader_fault_codes(ref_file, tmp_path):
    *_, path = ref_file
    raw = open(path, "rb").read()
    bad = tmp_path / "bad"
    b = bytearray(raw)
    b[len(b) // 2] ^= 0xFF                                     # flipped payload byte
    bad.write_bytes(bytes(b))
    assert _load_err(str(bad)) == "checksum-failure"
    bad.write_bytes(b"NOTANIDX" + raw[8:])
    assert _load_err(str(bad)) == "not-an-index"
    bad.write_bytes(raw[:8] + struct.pack("<I", 2) + raw[12:])
    assert _load_err(str(bad)) == "version-mismatch"
    bad.write_bytes(raw[: len(raw) - 7])
    assert _load_err(str(bad)) == "truncated-file"
    assert _load_err(str(tmp_path / "missing")) == "io-error"


@pytest.mark.gpu
def test_gpu_built_index_serializes_to_reference_bytes(ref_file, ref, tmp_path):
    p, c, kg, rix, path = ref_file
    dc = fg.DeviceCorpus(c)
    gix = fg.build_hybrid_index(dc, kg, degree=8, knn_k=16, seed=42, logical_cap=16)
    ours = str(tmp_path / "gpu.hybgrix")
    gix.serialize(ours)
    assert open(ours, "rb").read() == open(path, "rb").read()
    back = ref.index_deserialize(ours)                          # the reference reads our file
    want, got = ref.index_export(rix, c.n), ref.index_export(back, c.n)
    for key in ("semantic", "norm_order", "logical_ptr", "logical"):
        assert np.array_equal(want[key], got[key]), key


@pytest.mark.gpu
def test_reference_file_loads_into_hbm_and_searches_identically(ref_file, ref):
    p, c, kg, rix, path = ref_file
    gix = fg.HybridIndex.deserialize(path)
    want = ref.index_export(rix, c.n)
    got = gix.export()
    for key in ("semantic", "norm_order", "logical_ptr", "logical"):
        assert np.array_equal(want[key], got[key]), key
    q = synth.synth_queries(p, 40, beam_width=32)
    g, r = fg.batch_query(gix, q), ref.batch_query(rix, q)
    assert np.array_equal(g.doc_id, r.doc_id)
    assert np.array_equal(g.score.view(np.uint64), r.score.view(np.uint64))
