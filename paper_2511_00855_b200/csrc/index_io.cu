// index_io.cpp — the reference's binary index file `HYBGRIX1` v1
// (io.cpp:242-671) for the device index: a GPU-built index
// is written byte-for-byte as serialize_index would write it (so
// fusegraph::deserialize_index, the CLI `query`/`bench` and the CPU baseline
// at 10M load it), and a reference-written file loads straight into HBM.
//
// Format: magic "HYBGRIX1", u32 version 1, header (n, dense/learned/statistical
// dims u64; degree, knn_k, flags, default hops, logical cap u32; build seed
// u64), then sections {u32 id, u64 length, u64 FNV-1a of the payload,
// payload}, little-endian throughout, in the reference's order.  Errors use the
// reference's codes: not-an-index, version-mismatch, truncated-file,
// checksum-failure, io-error.
#include <cstring>
#include <fstream>
#include <map>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

#include "fg_cuda.hpp"
#include "index.hpp"

namespace fgb {
namespace {

constexpr char kMagic[8] = {'H', 'Y', 'B', 'G', 'R', 'I', 'X', '1'};
constexpr uint32_t kVersion = 1;
enum : uint32_t {
    kDocs = 1, kDense = 2, kLearned = 3, kStatistical = 4, kKeywords = 5, kEntities = 6,
    kSemantic = 7, kKeywordEdges = 8, kLogicalEdges = 9, kEntityMap = 10, kNormOrder = 11,
    kTriplets = 12
};
enum : uint32_t { kHasKeywordEdges = 1, kHasLogicalEdges = 2, kHasEntities = 4, kHasKg = 8 };

uint64_t fnv1a(const char* p, size_t len) {
    uint64_t h = 14695981039346656037ULL;
    for (size_t i = 0; i < len; ++i) {
        h ^= static_cast<unsigned char>(p[i]);
        h *= 1099511628211ULL;
    }
    return h;
}

struct Out {
    std::string b;
    void u32(uint32_t v) {
        char c[4];
        for (int i = 0; i < 4; ++i) c[i] = static_cast<char>((v >> (8 * i)) & 0xFF);
        b.append(c, 4);
    }
    void u64(uint64_t v) {
        char c[8];
        for (int i = 0; i < 8; ++i) c[i] = static_cast<char>((v >> (8 * i)) & 0xFF);
        b.append(c, 8);
    }
    void f32(float v) {
        uint32_t x;
        std::memcpy(&x, &v, 4);
        u32(x);
    }
};

void section(Out& file, uint32_t id, const Out& payload) {
    file.u32(id);
    file.u64(payload.b.size());
    file.u64(fnv1a(payload.b.data(), payload.b.size()));
    file.b += payload.b;
}

// encode_id_lists (io.cpp:338-346) of a CSR
void id_lists(Out& o, const uint64_t* ptr, const uint32_t* idx, uint64_t n) {
    o.u64(ptr[n] - ptr[0]);
    for (uint64_t i = 0; i < n; ++i) o.u32(static_cast<uint32_t>(ptr[i + 1] - ptr[i]));
    for (uint64_t i = 0; i < n; ++i)
        for (uint64_t j = ptr[i]; j < ptr[i + 1]; ++j) o.u32(idx[j]);
}

struct Reader {
    const std::string& s;
    size_t pos, end;
    void need(size_t k) const {
        if (pos + k > end) throw Error("truncated-file", "index file ends mid-record");
    }
    uint32_t u32() {
        need(4);
        uint32_t v = 0;
        for (int i = 0; i < 4; ++i) v |= static_cast<uint32_t>(static_cast<unsigned char>(s[pos + i])) << (8 * i);
        pos += 4;
        return v;
    }
    uint64_t u64() {
        need(8);
        uint64_t v = 0;
        for (int i = 0; i < 8; ++i) v |= static_cast<uint64_t>(static_cast<unsigned char>(s[pos + i])) << (8 * i);
        pos += 8;
        return v;
    }
    float f32() {
        const uint32_t x = u32();
        float v;
        std::memcpy(&v, &x, 4);
        return v;
    }
    uint8_t u8() {
        need(1);
        return static_cast<uint8_t>(s[pos++]);
    }
};

// decode_id_lists (io.cpp:348-361) into a CSR
void read_lists(Reader& r, uint64_t n, std::vector<uint64_t>& ptr, std::vector<uint32_t>& idx) {
    const uint64_t total = r.u64();
    std::vector<uint32_t> cnt(n);
    for (uint64_t i = 0; i < n; ++i) cnt[i] = r.u32();
    ptr.assign(n + 1, 0);
    for (uint64_t i = 0; i < n; ++i) ptr[i + 1] = ptr[i] + cnt[i];
    idx.resize(ptr[n]);
    for (auto& v : idx) v = r.u32();
    if (ptr[n] != total) throw Error("truncated-file", "id-list section count mismatch");
}

// The device corpus's sparse path as host CSR (padding stripped).
void sparse_host(const fg_corpus& c, bool learned, std::vector<uint64_t>& ptr, std::vector<uint32_t>& idx,
                 std::vector<float>& val) {
    const uint64_t n = c.n;
    std::vector<uint64_t> off(n);
    std::vector<uint32_t> nnz(n);
    (learned ? c.l_off : c.s_off).download(off.data(), n, c.stream);
    (learned ? c.l_nnz : c.s_nnz).download(nnz.data(), n, c.stream);
    const uint64_t total4 = learned ? c.l_nnz_total4 : c.s_nnz_total4;
    std::vector<uint32_t> pidx(total4 * 4);
    std::vector<float> pval(total4 * 4);
    (learned ? c.l_idx : c.s_idx).download(pidx.data(), total4 * 4, c.stream);
    (learned ? c.l_val : c.s_val).download(pval.data(), total4 * 4, c.stream);
    FGB_CUDA(cudaStreamSynchronize(c.stream));
    ptr.assign(n + 1, 0);
    for (uint64_t i = 0; i < n; ++i) ptr[i + 1] = ptr[i] + nnz[i];
    idx.resize(ptr[n]);
    val.resize(ptr[n]);
    for (uint64_t i = 0; i < n; ++i) {
        std::copy(pidx.begin() + off[i], pidx.begin() + off[i] + nnz[i], idx.begin() + ptr[i]);
        std::copy(pval.begin() + off[i], pval.begin() + off[i] + nnz[i], val.begin() + ptr[i]);
    }
}

// serialize_index (io.cpp:411-513)
std::string encode(const fg_index& ix) {
    const fg_corpus& c = *ix.corpus;
    const uint64_t n = c.n;
    const bool kw_edges = !ix.keyword_h.idx.empty();
    const bool logical = !ix.lg_h.empty();
    const bool entities = !c.entities.idx.empty();
    const bool has_kg = !ix.triplets.empty();
    Out f;
    f.b.append(kMagic, 8);
    f.u32(kVersion);
    f.u64(n);
    f.u64(c.dim);
    f.u64(c.learned_dim);
    f.u64(c.statistical_dim);
    f.u32(ix.degree);
    f.u32(ix.knn_k);
    f.u32((kw_edges ? kHasKeywordEdges : 0u) | (logical ? kHasLogicalEdges : 0u) |
          (entities ? kHasEntities : 0u) | (has_kg ? kHasKg : 0u));
    f.u32(ix.default_hops);
    f.u32(ix.logical_cap);
    f.u64(ix.seed);
    {
        Out s;
        for (uint64_t i = 0; i < n; ++i) {
            s.u64(c.doc_id[i]);
            s.b.push_back(c.deleted_h[i] ? 1 : 0);
        }
        section(f, kDocs, s);
    }
    {
        std::vector<float> dense(n * c.dstride);
        c.dense.download(dense.data(), n * c.dstride, c.stream);
        FGB_CUDA(cudaStreamSynchronize(c.stream));
        Out s;
        s.b.reserve(n * c.dim * 4);
        for (uint64_t i = 0; i < n; ++i)
            for (uint32_t j = 0; j < c.dim; ++j) s.f32(dense[i * c.dstride + j]);
        section(f, kDense, s);
    }
    for (int p = 0; p < 2; ++p) {  // encode_sparse_column (io.cpp:363-381)
        std::vector<uint64_t> ptr;
        std::vector<uint32_t> idx;
        std::vector<float> val;
        sparse_host(c, p == 0, ptr, idx, val);
        Out s;
        s.u64(ptr[n]);
        for (uint64_t i = 0; i < n; ++i) s.u32(static_cast<uint32_t>(ptr[i + 1] - ptr[i]));
        for (uint64_t j = 0; j < ptr[n]; ++j) {
            s.u32(idx[j]);
            s.f32(val[j]);
        }
        section(f, p == 0 ? kLearned : kStatistical, s);
    }
    {
        Out s;
        id_lists(s, c.keywords.ptr.data(), c.keywords.idx.data(), n);
        section(f, kKeywords, s);
    }
    if (entities) {
        Out s;
        id_lists(s, c.entities.ptr.data(), c.entities.idx.data(), n);
        section(f, kEntities, s);
    }
    {
        std::vector<uint64_t> ptr(n + 1);
        for (uint64_t i = 0; i <= n; ++i) ptr[i] = i * ix.degree;
        Out s;
        id_lists(s, ptr.data(), ix.semantic_h.data(), n);
        section(f, kSemantic, s);
    }
    if (kw_edges) {
        Out s;
        id_lists(s, ix.keyword_h.ptr.data(), ix.keyword_h.idx.data(), n);
        section(f, kKeywordEdges, s);
    }
    if (logical) {
        Out s;
        s.u64(ix.lg_ptr_h[n]);
        for (uint64_t i = 0; i < n; ++i) s.u32(static_cast<uint32_t>(ix.lg_ptr_h[i + 1] - ix.lg_ptr_h[i]));
        for (uint64_t e = 0; e < ix.lg_ptr_h[n] * 4; ++e) s.u32(ix.lg_h[e]);
        section(f, kLogicalEdges, s);
    }
    if (entities) {
        Out s;
        s.u32(static_cast<uint32_t>(ix.entity_map.size()));
        for (const auto& [e, nodes] : ix.entity_map) {
            s.u32(e);
            s.u32(static_cast<uint32_t>(nodes.size()));
            for (uint32_t v : nodes) s.u32(v);
        }
        section(f, kEntityMap, s);
    }
    {
        Out s;
        for (uint32_t v : ix.norm_order_h) s.u32(v);
        section(f, kNormOrder, s);
    }
    if (has_kg) {
        Out s;
        s.u64(ix.triplets.size() / 3);
        for (uint32_t v : ix.triplets) s.u32(v);
        section(f, kTriplets, s);
    }
    return std::move(f.b);
}

}  // namespace
}  // namespace fgb

using namespace fgb;

extern "C" {

int fg_index_serialize(const fg_index* ix, const char* path, uint64_t* bytes) {
    return guarded([&] {
        if (!ix || !path) throw Error("invalid-argument", "null pointer");
        FGB_CUDA(cudaSetDevice(ix->corpus->device));
        const std::string file = encode(*ix);
        std::ofstream out(path, std::ios::binary | std::ios::trunc);
        if (!out) throw Error("io-error", std::string("cannot open ") + path + " for writing");
        out.write(file.data(), static_cast<std::streamsize>(file.size()));
        if (!out) throw Error("io-error", std::string("failed writing ") + path);
        if (bytes) *bytes = file.size();
    });
}

int fg_index_deserialize(const char* path, int device, fg_corpus** corpus_out, fg_index** index_out) {
    return guarded([&] {
        if (!path || !corpus_out || !index_out) throw Error("invalid-argument", "null pointer");
        std::ifstream in(path, std::ios::binary);
        if (!in) throw Error("io-error", std::string("cannot open ") + path);
        std::ostringstream buf;
        buf << in.rdbuf();
        const std::string bytes = buf.str();
        if (bytes.size() < 12 || std::memcmp(bytes.data(), kMagic, 8) != 0)
            throw Error("not-an-index", std::string(path) + " lacks the index magic");
        Reader h{bytes, 8, bytes.size()};
        const uint32_t version = h.u32();
        if (version != kVersion)
            throw Error("version-mismatch",
                        "index format " + std::to_string(version) + ", expected " + std::to_string(kVersion));
        const uint64_t n = h.u64();
        const uint64_t dense_dim = h.u64(), learned_dim = h.u64(), statistical_dim = h.u64();
        const uint32_t degree = h.u32(), knn_k = h.u32(), flags = h.u32(), hops = h.u32(), lcap = h.u32();
        const uint64_t seed = h.u64();

        std::vector<uint64_t> doc_id(n);
        std::vector<uint8_t> deleted(n);
        std::vector<float> dense;
        std::vector<uint64_t> sp_ptr[2], kw_ptr, ent_ptr, sem_ptr, kwe_ptr, lg_ptr(n + 1, 0);
        std::vector<uint32_t> sp_idx[2], kw_idx, ent_idx, sem_idx, kwe_idx, lg, norm, trip;
        std::vector<float> sp_val[2];
        std::map<uint32_t, std::vector<uint32_t>> emap;
        uint32_t seen = 0;
        size_t pos = h.pos;
        while (pos < bytes.size()) {
            Reader hd{bytes, pos, bytes.size()};
            const uint32_t id = hd.u32();
            const uint64_t len = hd.u64();
            const uint64_t sum = hd.u64();
            const size_t start = hd.pos;
            if (start + len > bytes.size())
                throw Error("truncated-file", "section " + std::to_string(id) + " extends past end of file");
            if (fnv1a(bytes.data() + start, len) != sum)
                throw Error("checksum-failure", "section " + std::to_string(id) + " is corrupted");
            Reader r{bytes, start, start + len};
            switch (id) {
                case kDocs:
                    for (uint64_t i = 0; i < n; ++i) {
                        doc_id[i] = r.u64();
                        deleted[i] = r.u8() != 0;
                    }
                    break;
                case kDense:
                    dense.resize(n * dense_dim);
                    for (auto& v : dense) v = r.f32();
                    break;
                case kLearned:
                case kStatistical: {
                    const int p = id == kLearned ? 0 : 1;
                    r.u64();
                    std::vector<uint32_t> cnt(n);
                    for (auto& x : cnt) x = r.u32();
                    sp_ptr[p].assign(n + 1, 0);
                    for (uint64_t i = 0; i < n; ++i) sp_ptr[p][i + 1] = sp_ptr[p][i] + cnt[i];
                    sp_idx[p].resize(sp_ptr[p][n]);
                    sp_val[p].resize(sp_ptr[p][n]);
                    for (uint64_t j = 0; j < sp_ptr[p][n]; ++j) {
                        sp_idx[p][j] = r.u32();
                        sp_val[p][j] = r.f32();
                    }
                    break;
                }
                case kKeywords: read_lists(r, n, kw_ptr, kw_idx); break;
                case kEntities: read_lists(r, n, ent_ptr, ent_idx); break;
                case kSemantic: read_lists(r, n, sem_ptr, sem_idx); break;
                case kKeywordEdges: read_lists(r, n, kwe_ptr, kwe_idx); break;
                case kLogicalEdges: {
                    r.u64();
                    for (uint64_t i = 0; i < n; ++i) lg_ptr[i + 1] = lg_ptr[i] + r.u32();
                    lg.resize(lg_ptr[n] * 4);
                    for (auto& v : lg) v = r.u32();
                    break;
                }
                case kEntityMap: {
                    const uint32_t keys = r.u32();
                    for (uint32_t i = 0; i < keys; ++i) {
                        const uint32_t e = r.u32();
                        const uint32_t cnt = r.u32();
                        auto& nodes = emap[e];
                        nodes.resize(cnt);
                        for (auto& v : nodes) v = r.u32();
                    }
                    break;
                }
                case kNormOrder:
                    norm.resize(n);
                    for (auto& v : norm) v = r.u32();
                    break;
                case kTriplets: {
                    const uint64_t cnt = r.u64();
                    trip.resize(cnt * 3);
                    for (auto& v : trip) v = r.u32();
                    break;
                }
                default:
                    throw Error("version-mismatch", "unknown section id " + std::to_string(id));
            }
            seen |= 1u << id;
            pos = start + len;
        }
        const uint32_t required = (1u << kDocs) | (1u << kDense) | (1u << kLearned) | (1u << kStatistical) |
                                  (1u << kKeywords) | (1u << kSemantic) | (1u << kNormOrder);
        if ((seen & required) != required) throw Error("truncated-file", "index file is missing required sections");
        if ((flags & kHasKeywordEdges) && !(seen & (1u << kKeywordEdges)))
            throw Error("truncated-file", "keyword edge section missing");
        if ((flags & kHasLogicalEdges) && !(seen & (1u << kLogicalEdges)))
            throw Error("truncated-file", "logical edge section missing");
        if ((flags & kHasEntities) && !(seen & (1u << kEntityMap)))
            throw Error("truncated-file", "entity sections missing");
        if ((flags & kHasKg) && !(seen & (1u << kTriplets)))
            throw Error("truncated-file", "knowledge graph section missing");
        for (uint64_t i = 0; i < n; ++i)
            if (sem_ptr[i + 1] - sem_ptr[i] != degree)
                throw Error("invariant-violation", "semantic list of node " + std::to_string(i) + " is not degree long");
        if (ent_ptr.empty()) ent_ptr.assign(n + 1, 0);

        fg_corpus_view v{};
        v.n = n;
        v.dense_dim = static_cast<uint32_t>(dense_dim);
        v.learned_dim = static_cast<uint32_t>(learned_dim);
        v.statistical_dim = static_cast<uint32_t>(statistical_dim);
        v.dense = dense.data();
        v.learned = fg_sparse_view{sp_ptr[0].data(), sp_idx[0].data(), sp_val[0].data()};
        v.statistical = fg_sparse_view{sp_ptr[1].data(), sp_idx[1].data(), sp_val[1].data()};
        v.keywords = fg_list_view{kw_ptr.data(), kw_idx.data()};
        v.entities = fg_list_view{ent_ptr.data(), ent_idx.data()};
        v.doc_id = doc_id.data();
        v.deleted = deleted.data();
        fg_corpus* c = nullptr;
        if (fg_corpus_upload(&v, device, &c) != FG_OK) throw Error(fg_last_error_code(), fg_last_error_message());
        std::unique_ptr<fg_corpus, int (*)(fg_corpus*)> cg(c, fg_corpus_free);
        std::vector<uint32_t> ks(trip.size() / 3), kr(ks.size()), kt(ks.size());
        for (size_t i = 0; i < ks.size(); ++i) {
            ks[i] = trip[3 * i];
            kr[i] = trip[3 * i + 1];
            kt[i] = trip[3 * i + 2];
        }
        const fg_kg_view kg{ks.size(), ks.data(), kr.data(), kt.data()};
        if (kwe_ptr.empty()) kwe_ptr.assign(n + 1, 0);
        fg_graph_view gv{};
        gv.degree = degree;
        gv.semantic = sem_idx.data();
        gv.keyword = fg_list_view{kwe_ptr.data(), kwe_idx.data()};
        gv.logical_ptr = lg_ptr.data();
        gv.logical = lg.data();
        gv.norm_order = norm.data();
        fg_index* ix = nullptr;
        if (fg_index_create(c, &kg, &gv, &ix) != FG_OK) throw Error(fg_last_error_code(), fg_last_error_message());
        ix->knn_k = knn_k;
        ix->default_hops = hops;
        ix->logical_cap = lcap;
        ix->seed = seed;
        ix->entity_map = std::move(emap);  // as stored (the reference trusts the file)
        *corpus_out = cg.release();
        *index_out = ix;
    });
}

}  // extern "C"
