/*
 * fg_b200.h — C-ABI of the B200-native hybrid-search hot path.
 *
 * This is the drop-in boundary under the reference's C++ API
 * (/root/reference/proj/include/fusegraph/ headers, "fusegraph"): every entry
 * point below replaces one reference function on the hot path and is cited
 * as `file:line` of the reference interface it stands in for.  The reference
 * C++ shim that forwards `fusegraph::` calls to these symbols is shown in
 * INTEGRATION.md.
 *
 * Conventions
 *  - Plain pointers and sizes only; no torch / STL types cross the boundary.
 *  - Every function returns FG_OK (0) or FG_ERR (1).  On FG_ERR the calling
 *    thread's last error carries the reference's machine code ("dim-mismatch",
 *    "invalid-k", "corpus-too-small", ...) and the full message, formatted as
 *    the reference's `fusegraph::Error::what()` ("<code>: <message>",
 *    error.hpp:11-20).  Read it with fg_last_error_code()/_message().
 *  - Node ids are positions in the corpus (types.hpp:117-118); doc ids are the
 *    external 64-bit identifiers.
 *  - Scores are fp64 similarities (types.hpp:15); distance = -score.
 *  - All compute runs on the GPU.  There is no CPU fallback: without a
 *    CUDA device every compute entry point fails with "no-cuda-device".
 */
#ifndef FG_B200_H
#define FG_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FG_ABI_VERSION 1
#define FG_OK 0
#define FG_ERR 1

/* Bits of fg_search_results.warnings (search.hpp:37, search.cpp:206,271). */
#define FG_WARN_ENTITY_FALLBACK 1u
#define FG_WARN_KEYWORD_SHORTFALL 2u

/* ------------------------------------------------------------------------ */
/* Flat, caller-owned views                                                  */
/* ------------------------------------------------------------------------ */

/* One sparse path for `rows` rows in CSR form (SparseVector, types.hpp:28-34):
 * row r owns entries [ptr[r], ptr[r+1]); indices strictly ascending per row.
 * ptr == NULL means every row is empty. */
typedef struct fg_sparse_view {
    const uint64_t* ptr; /* rows + 1 */
    const uint32_t* idx;
    const float* val;
} fg_sparse_view;

/* A sorted-id list per row (keywords, entities, required keywords). */
typedef struct fg_list_view {
    const uint64_t* ptr; /* rows + 1, NULL = all empty */
    const uint32_t* idx;
} fg_list_view;

/* DocumentStore (types.hpp:119-133) as structure-of-arrays. */
typedef struct fg_corpus_view {
    uint64_t n;
    uint32_t dense_dim;
    uint32_t learned_dim;     /* vocabulary bounds (informational) */
    uint32_t statistical_dim;
    const float* dense;       /* n * dense_dim, row-major */
    fg_sparse_view learned;
    fg_sparse_view statistical;
    fg_list_view keywords;    /* ptr == NULL: the statistical support (corpus.cpp:116) */
    fg_list_view entities;    /* sorted unique per doc */
    const uint64_t* doc_id;   /* NULL: doc_id = node */
    const uint8_t* deleted;   /* NULL: nothing deleted */
} fg_corpus_view;

/* Weights (types.hpp:49-54). */
typedef struct fg_weights {
    float dense;
    float learned;
    float statistical;
    float entity;
} fg_weights;

/* A batch of QuerySpec (types.hpp:70-78), raw (pre-weighting) vectors. */
typedef struct fg_query_view {
    uint64_t count;
    uint32_t dense_dim;
    const float* dense;             /* count * dense_dim */
    fg_sparse_view learned;
    fg_sparse_view statistical;
    const fg_weights* weights;      /* count */
    fg_list_view required_keywords; /* sorted per query */
    fg_list_view entities;          /* sorted per query */
    const uint32_t* k;              /* count (NULL: 10) */
    const uint32_t* beam_width;     /* count (NULL: 64) */
    const uint32_t* max_entity_hops;/* count (NULL: 2) */
} fg_query_view;

/* KnowledgeGraph triplets (types.hpp:80-113). */
typedef struct fg_kg_view {
    uint64_t count;
    const uint32_t* source;
    const uint32_t* relation;
    const uint32_t* target;
} fg_kg_view;

/* KnnGraph (knn_graph.hpp:26-39) as fixed-width arrays, caller-owned:
 * row u holds exactly k entries sorted by (score desc, id asc). */
typedef struct fg_knn_lists {
    uint64_t n;
    uint32_t k;
    uint32_t* ids;    /* n * k */
    double* scores;   /* n * k */
    uint8_t* fresh;   /* n * k */
} fg_knn_lists;

typedef struct fg_knn_params { /* KnnBuildParams, knn_graph.hpp:41-48 */
    uint32_t k;
    uint32_t max_iterations;
    double convergence;
    uint64_t seed;
} fg_knn_params;

typedef struct fg_refine_params { /* RefineParams, refine.hpp:41-48 */
    uint32_t degree;
    int per_neighbour_keyword_check;
} fg_refine_params;

/* RefinedEdges (refine.hpp:51-54), caller-owned fixed-capacity arrays. */
typedef struct fg_refined {
    uint32_t* semantic;       /* n * degree */
    uint32_t keyword_cap;     /* >= knn k */
    uint32_t* keyword;        /* n * keyword_cap, recycled ids in order */
    uint32_t* keyword_count;  /* n */
} fg_refined;

/* RefineTrace (refine.hpp:56-62); every pointer may be NULL. */
typedef struct fg_refine_trace {
    uint32_t* ordered_ids;    /* n * k, ranked candidates */
    double* ordered_scores;   /* n * k */
    uint32_t* detours;        /* n * k */
    uint32_t* kept;           /* n * degree */
    uint32_t* kept_count;     /* n */
} fg_refine_trace;

typedef struct fg_build_params { /* BuildParams, index.hpp:21-30 */
    uint32_t degree;
    uint32_t knn_k;
    uint32_t knn_iterations;
    uint64_t seed;
    uint32_t logical_cap;
    uint32_t default_entity_hops;
    int per_neighbour_keyword_check;
} fg_build_params;

/* Edge tables of a HybridIndex (index.hpp:33-52). */
typedef struct fg_graph_view {
    uint32_t degree;
    const uint32_t* semantic;     /* n * degree */
    fg_list_view keyword;         /* per node, reach order (not sorted) */
    const uint64_t* logical_ptr;  /* n + 1 */
    const uint32_t* logical;      /* 4 u32 per edge: source, relation, target, via */
    const uint32_t* norm_order;   /* n */
} fg_graph_view;

typedef struct fg_search_opts { /* SearchOptions, search.hpp:45-49 */
    uint32_t entry_count;
    int conjunctive_filter;
} fg_search_opts;

/* Per-query SearchResult (search.hpp:31-43) in caller-owned arrays. */
typedef struct fg_search_results {
    uint32_t hit_stride;   /* >= max k of the batch */
    uint64_t* doc_id;      /* count * hit_stride */
    uint32_t* node;        /* count * hit_stride */
    double* score;         /* count * hit_stride */
    uint32_t* hit_count;   /* count */
    uint64_t* expanded;    /* count (may be NULL) */
    uint64_t* scored;      /* count, distinct nodes scored (may be NULL) */
    uint32_t* warnings;    /* count, FG_WARN_* bits (may be NULL) */
    char* errors;          /* count * error_stride, "" when ok (may be NULL) */
    uint32_t error_stride;
} fg_search_results;

/* SynthParams (synth.hpp:19-45). */
typedef struct fg_synth_params {
    uint32_t docs, dense_dim, clusters;
    float cluster_spread;
    uint32_t learned_vocab, learned_nnz, statistical_vocab, statistical_nnz;
    double zipf_exponent;
    uint32_t entity_vocab;
    double entity_rate;
    uint32_t max_entities_per_doc, kg_triplets, relation_vocab, chains, answers_per_chain;
    uint64_t seed;
} fg_synth_params;

typedef struct fg_host_corpus fg_host_corpus; /* generator output, library-owned */
typedef struct fg_corpus fg_corpus;           /* device mirror of a DocumentStore */
typedef struct fg_index fg_index;             /* device-resident HybridIndex */
typedef struct fg_comm fg_comm;               /* NCCL communicator of a sharded build */

/* ------------------------------------------------------------------------ */
/* Errors and devices                                                         */
/* ------------------------------------------------------------------------ */

int fg_abi_version(void);
const char* fg_last_error_code(void);    /* "" when none */
const char* fg_last_error_message(void); /* "<code>: <message>" */
int fg_device_count(int* count);

/* ------------------------------------------------------------------------ */
/* Synthetic data: bit-identical to generate_corpus / random_query_vector /   */
/* random_simplex_weights (synth.hpp:61-67, synth.cpp:140-222), generated     */
/* straight into CSR on host threads (no AoS).                               */
/* ------------------------------------------------------------------------ */

int fg_synth_generate(const fg_synth_params* p, unsigned threads, fg_host_corpus** out);
/* Views into the generated arrays (valid until fg_host_corpus_free). */
int fg_host_corpus_view(const fg_host_corpus* h, fg_corpus_view* corpus, fg_kg_view* kg,
                        uint64_t* chain_count);
/* Chain c: {e0,e1,e2}, seed/bridge doc, answers (answers_per_chain), and the
 * planted query vector (dense_dim floats + learned/statistical CSR of one row). */
int fg_host_corpus_chain(const fg_host_corpus* h, uint64_t c, uint32_t ent[3], uint64_t docs[2],
                         uint64_t* answers, float* dense, uint32_t* learned_nnz,
                         uint32_t* learned_idx, float* learned_val, uint32_t* stat_nnz,
                         uint32_t* stat_idx, float* stat_val);
int fg_host_corpus_free(fg_host_corpus* h);

/* `count` queries from SplitMix64(mix_seed(seed, stream)), each drawn as
 * random_query_vector then (if with_weights) random_simplex_weights, as the
 * CLI does (fusegraph_cli.cpp:184-194).  Output arrays are caller-owned:
 * dense count*dense_dim, learned/statistical exactly count*nnz entries
 * (fixed nnz per query), weights count. */
int fg_synth_queries(const fg_synth_params* p, uint64_t stream, uint64_t count,
                     int with_weights, float* dense, uint32_t* learned_idx, float* learned_val,
                     uint32_t* stat_idx, float* stat_val, fg_weights* weights);

/* ------------------------------------------------------------------------ */
/* Device corpus (the DocumentStore on HBM)                                  */
/* ------------------------------------------------------------------------ */

/* Packs the corpus into the device row-blob layout and computes the cached
 * squared norms on the GPU (finalize_fused, types.cpp:74-79).  Validates the
 * structural contract of validate_corpus (corpus.cpp:39-84) for what the GPU
 * relies on: uniform dense dim, ascending sparse indices. */
int fg_corpus_upload(const fg_corpus_view* view, int device, fg_corpus** out);
int fg_corpus_free(fg_corpus* c);
int fg_corpus_size(const fg_corpus* c, uint64_t* n, uint32_t* dense_dim);
int fg_corpus_sqnorm(const fg_corpus* c, double* out); /* n values */
/* mark_delete (update.hpp:38) flag mirror. */
int fg_corpus_set_deleted(fg_corpus* c, const uint8_t* flags);

/* ------------------------------------------------------------------------ */
/* Hybrid distance kernel (K1)                                               */
/* ------------------------------------------------------------------------ */

/* build_query_vector (corpus.hpp:34, corpus.cpp:86-103) for query i of a batch:
 * dense_out dense_dim floats; sparse outputs sized as the input row; the
 * *_nnz outputs are 0 for a zero-weight path.  Host arithmetic is the
 * reference's fp32 product; the GPU kernels apply the identical product. */
int fg_build_query_vector(const fg_query_view* q, uint64_t i, float* dense_out,
                          uint32_t* learned_nnz, float* learned_val, uint32_t* stat_nnz,
                          float* stat_val, double* squared_norm);

/* batch_scores (scoring.hpp:32-36): hybrid_score of weighted query qi against
 * each node in ids, in input order. */
int fg_batch_scores(const fg_corpus* c, const fg_query_view* q, uint64_t qi, const uint32_t* ids,
                    uint64_t m, double* out);

/* hybrid_score(doc a, doc b) under unit weights for m pairs (the pair_score of
 * knn_graph.cpp:20-22 and candidate_pair_scores, refine.cpp:11-23). */
int fg_pair_scores(const fg_corpus* c, const uint32_t* a, const uint32_t* b, uint64_t m,
                   double* out);

/* ------------------------------------------------------------------------ */
/* Graph construction (K3 NN-Descent, K4 refinery)                          */
/* ------------------------------------------------------------------------ */

/* init_random_graph (knn_graph.hpp:52-53). out->n == corpus n, out->k == k. */
int fg_knn_init(const fg_corpus* c, uint32_t k, uint64_t seed, fg_knn_lists* out);
/* nn_descent_iterate (knn_graph.hpp:56): one double-buffered pass in place. */
int fg_knn_iterate(const fg_corpus* c, fg_knn_lists* lists, uint64_t* changed);
/* build_knn_graph (knn_graph.hpp:59).  The caller allocates n*params->k slots;
 * out->k receives the (possibly clamped) k. passes may be NULL. */
int fg_knn_build(const fg_corpus* c, const fg_knn_params* params, fg_knn_lists* out,
                 uint32_t* passes);

/* refine_graph (refine.hpp:87-89). trace may be NULL. */
int fg_refine(const fg_corpus* c, const fg_knn_lists* knn, const fg_refine_params* params,
              fg_refined* out, fg_refine_trace* trace);

/* ------------------------------------------------------------------------ */
/* Index (L4)                                                                */
/* ------------------------------------------------------------------------ */

/* build_hybrid_index (index.hpp:60-61).  The index keeps a reference to the
 * corpus, which must outlive it.  Logical edges (logical.cpp:17-68) and the
 * norm order (index.cpp:12-23) are derived as in the reference. */
int fg_index_build(fg_corpus* c, const fg_kg_view* kg, const fg_build_params* params,
                   fg_index** out);
/* Wraps an index built elsewhere (e.g. loaded by deserialize_index, io.hpp:71)
 * without rebuilding; degree/keyword/logical tables are uploaded as given. */
int fg_index_create(fg_corpus* c, const fg_kg_view* kg, const fg_graph_view* graph,
                    fg_index** out);
int fg_index_sizes(const fg_index* ix, uint32_t* degree, uint64_t* keyword_total,
                   uint64_t* logical_total);
/* Host copies of the edge tables (each pointer may be NULL). */
int fg_index_export(const fg_index* ix, uint32_t* semantic, uint64_t* keyword_ptr,
                    uint32_t* keyword_idx, uint64_t* logical_ptr, uint32_t* logical,
                    uint32_t* norm_order);
/* Seconds spent in the last fg_index_build, split by stage (may be NULL):
 * [0] knn, [1] refine, [2] logical+entity map, [3] norm order, [4] total. */
int fg_index_build_times(const fg_index* ix, double* seconds5);
/* NN-Descent totals of fg_index_build: {passes, candidate pair scores (the
 * sum over passes and nodes of S_u, knn_graph.cpp:122-131), dense rows read
 * after the certified screening, device microseconds of the pass kernels};
 * zeros for other builds.  Feeds the build roofline of bench.py. */
int fg_index_build_stats(const fg_index* ix, uint64_t* stats4);
/* The same counters followed by {candidates bounded by the pass-1 sparse
 * sketches, candidates those bounds rejected before their postings were
 * read}; the first `count` of the 6 (zeros past them). */
int fg_index_build_stats_ex(const fg_index* ix, uint64_t* stats, uint32_t count);
int fg_index_free(fg_index* ix);

/* InsertParams (update.hpp:22-28). */
typedef struct fg_insert_params {
    uint32_t knn_k;                 /* candidate width; 0: the build's knn_k */
    uint32_t nn_descent_iterations; /* batch-local NN-Descent passes (10) */
    uint32_t threads;               /* accepted for API parity; the GPU ignores it */
} fg_insert_params;

/* insert_batch (update.hpp:33-34, update.cpp:33-197): appends `docs` to the
 * index's corpus and links them exactly as the reference does (beam-search
 * candidates over the current graph, NN-Descent among the batch, per-node
 * refinery, batch-local reverse half, weakest-reverse-slot replacement on
 * existing nodes, norm order rebuilt).  Validation happens first and leaves
 * the index untouched on error (duplicate-id, dim-mismatch, nonfinite-value,
 * unsorted-sparse, zero-sparse-value, invalid-k, corpus-too-small). */
int fg_index_insert(fg_index* ix, const fg_corpus_view* docs, const fg_insert_params* params);

/* The reference's binary index file HYBGRIX1 v1 (io.hpp:63-71, io.cpp:242-671,
 * SURVEY 8(f2)).  fg_index_serialize writes exactly the bytes
 * fusegraph::serialize_index writes for the same index (the reference's
 * deserialize_index, CLI `query`/`bench` load it); fg_index_deserialize loads
 * a reference-written file into a new device corpus + index (errors:
 * not-an-index, version-mismatch, truncated-file, checksum-failure, io-error). */
int fg_index_serialize(const fg_index* ix, const char* path, uint64_t* bytes);
int fg_index_deserialize(const char* path, int device, fg_corpus** corpus, fg_index** index);

/* ------------------------------------------------------------------------ */
/* Multi-GPU construction: vertex-range sharding              */
/* ------------------------------------------------------------------------ */

/* One process per GPU.  Rank 0 creates the id, the caller broadcasts it (any
 * host channel, e.g. torch.distributed), every rank then calls fg_comm_init.
 * NCCL is loaded at run time (libnccl.so.2). */
#define FG_COMM_ID_BYTES 128
int fg_comm_unique_id(uint8_t* id /* FG_COMM_ID_BYTES */);
int fg_comm_init(int nranks, int rank, const uint8_t* id, int device, fg_comm** out);
int fg_comm_free(fg_comm* comm);

/* A communicator whose collectives run through caller callbacks on host
 * buffers (e.g. torch.distributed gloo) instead of NCCL: the same sharded
 * build, each collective staged device -> host -> callback -> device.  For
 * hosts without NCCL peers and for multi-process tests of the sharding with
 * several ranks on one GPU.  all_gather: `send` holds this rank's `bytes`,
 * `recv` receives every rank's in rank order (nranks * bytes); sum_u64: `x`
 * (`count` values) is replaced by the sum over ranks.  Return 0 on success. */
typedef int (*fg_host_all_gather_fn)(void* ctx, const void* send, void* recv, uint64_t bytes);
typedef int (*fg_host_sum_u64_fn)(void* ctx, uint64_t* x, uint64_t count);
int fg_comm_init_host(int nranks, int rank, int device, fg_host_all_gather_fn all_gather,
                      fg_host_sum_u64_fn sum_u64, void* ctx, fg_comm** out);

/* build_hybrid_index (index.hpp:60-61) sharded by vertex range: rank r runs
 * the NN-Descent passes and the per-node refinery for nodes
 * [r*ceil(n/G), (r+1)*ceil(n/G)), all-gathering each pass's lists and the
 * refined lists over NCCL; merge_reverse_edges, logical edges and the norm
 * order are replicated.  The index is identical on every rank and identical
 * to fg_index_build's (the passes are double-buffered, knn_graph.cpp:91).
 * comm == NULL with sim_ranks = G > 1 runs all G ranges in this process (no
 * collective) — the partition logic on one GPU, for parity tests. */
int fg_index_build_sharded(fg_corpus* c, const fg_kg_view* kg, const fg_build_params* params,
                           fg_comm* comm, uint32_t sim_ranks, fg_index** out);

/* ------------------------------------------------------------------------ */
/* Batched beam search (K5) and exhaustive truth (K6)                       */
/* ------------------------------------------------------------------------ */

/* batch_query (search.hpp:86-88) — one query per result row; per-query
 * validation errors are captured into out->errors like search.cpp:286-290.
 * `out` rows are filled for every query. */
int fg_batch_query(const fg_index* ix, const fg_query_view* q, const fg_search_opts* opts,
                   fg_search_results* out);

/* Same, with queries already resident on the device in the view's layout is
 * not part of the ABI: the host view is copied every call (that copy is in
 * the end-to-end number). */

/* brute_force_topk (eval.hpp:20-21) for every query of the batch. */
int fg_brute_force_topk(const fg_corpus* c, const fg_query_view* q, fg_search_results* out);

/* Device time (ms, CUDA events) of the last fg_batch_query's search kernel,
 * and the number of kernel launches it issued. */
int fg_last_search_stats(const fg_index* ix, double* kernel_ms, uint64_t* launches);

/* Name of the kernel the last fg_batch_query ran ("search_plain_kernel",
 * "search_hybrid_kernel" or "search_kernel"; "" before the first call). */
int fg_last_search_kernel(const fg_index* ix, const char** name);

/* Diagnostics of the refinery's tensor-core candidate Gram (refine.cu,
 * gram_tc_*; replaces the dense half of candidate_pair_scores,
 * refine.cpp:11-23, with a certified split-bf16 tcgen05 product): pairs
 * scored, pairs re-scored exactly because they fell within the error bound of
 * a decision threshold, and (FGB_REFINE_TC_CHECK=1) the largest measured
 * |approx - exact| / (|x||y|).  Counting is on while FGB_REFINE_TC_STATS=1
 * or FGB_REFINE_TC_CHECK=1; reset != 0 zeroes the counters after reading. */
int fg_refine_tc_stats(uint64_t* pairs, uint64_t* resolved, double* max_rel_err, int reset);

#ifdef __cplusplus
} /* extern "C" */
#endif

#endif /* FG_B200_H */
