// Host pieces of the mpic:: API: config, hashing, KvTensor, the GEMM shims, and the glue
// to the C ABI (device.h).
#include "device.h"

#include "mpic/config.h"
#include "mpic/hash.h"
#include "mpic/matmul.h"
#include "mpic/tensor.h"

#include <openssl/evp.h>
#include <zlib.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <vector>

namespace mpic {

// ---- config (proj/src/config.cpp:12-47 semantics) -------------------------------------
void ModelConfig::validate() const {
    const mpic_model_config c = b200::to_c(*this);
    b200::check(mpic_config_validate(&c));
}

uint64_t ModelConfig::fingerprint() const {
    const mpic_model_config c = b200::to_c(*this);
    return mpic_config_fingerprint(&c);
}

// ---- hashing --------------------------------------------------------------------------
Hash256 sha256(std::span<const uint8_t> bytes) {
    Hash256 out{};
    unsigned int n = 0;
    EVP_MD_CTX* ctx = EVP_MD_CTX_new();
    const bool ok = ctx && EVP_DigestInit_ex(ctx, EVP_sha256(), nullptr) == 1 &&
                    EVP_DigestUpdate(ctx, bytes.data(), bytes.size()) == 1 &&
                    EVP_DigestFinal_ex(ctx, out.data(), &n) == 1 && n == out.size();
    EVP_MD_CTX_free(ctx);
    if (!ok) throw io_error("sha256 failed");
    return out;
}

std::string hash_to_hex(const Hash256& h) {
    static constexpr char kHex[] = "0123456789abcdef";
    std::string s(64, '0');
    for (size_t i = 0; i < h.size(); ++i) {
        s[2 * i] = kHex[h[i] >> 4];
        s[2 * i + 1] = kHex[h[i] & 15];
    }
    return s;
}

Hash256 hash_from_hex(std::string_view hex) {
    if (hex.size() != 64) throw validation_error("content hash must be 64 hex characters");
    auto val = [](char c) -> int {
        if (c >= '0' && c <= '9') return c - '0';
        if (c >= 'a' && c <= 'f') return c - 'a' + 10;
        if (c >= 'A' && c <= 'F') return c - 'A' + 10;
        return -1;
    };
    Hash256 h{};
    for (size_t i = 0; i < 32; ++i) {
        const int hi = val(hex[2 * i]), lo = val(hex[2 * i + 1]);
        if (hi < 0 || lo < 0) throw validation_error("content hash contains non-hex characters");
        h[i] = static_cast<uint8_t>(hi * 16 + lo);
    }
    return h;
}

uint32_t crc32_of(std::span<const uint8_t> bytes) {
    uLong c = crc32(0L, Z_NULL, 0);
    // zlib takes 32-bit lengths: feed large payloads in pieces
    size_t off = 0;
    while (off < bytes.size()) {
        const size_t n = std::min<size_t>(bytes.size() - off, size_t(1) << 30);
        c = crc32(c, bytes.data() + off, static_cast<uInt>(n));
        off += n;
    }
    return static_cast<uint32_t>(c);
}

// ---- KvTensor -------------------------------------------------------------------------
void KvTensor::resize_tokens(uint32_t new_tokens) {
    if (new_tokens == n_tokens) return;
    const size_t row = row_size();
    const size_t keep = size_t(std::min(n_tokens, new_tokens)) * row;
    std::vector<float> nk(size_t(n_layers) * new_tokens * row, 0.0f), nv(nk.size(), 0.0f);
    for (uint32_t l = 0; l < n_layers; ++l) {
        std::copy_n(k.data() + size_t(l) * n_tokens * row, keep, nk.data() + size_t(l) * new_tokens * row);
        std::copy_n(v.data() + size_t(l) * n_tokens * row, keep, nv.data() + size_t(l) * new_tokens * row);
    }
    k.swap(nk);
    v.swap(nv);
    n_tokens = new_tokens;
}

bool KvTensor::all_finite() const {
    auto fin = [](const std::vector<float>& a) {
        return std::all_of(a.begin(), a.end(), [](float x) { return std::isfinite(x); });
    };
    return fin(k) && fin(v);
}

// ---- GEMM shims (run on the device, fp32 SIMT) ----------------------------------------
namespace {
int g_threads = 0;

void device_gemm_nt(int m, int n, int k, const float* a, int lda, const float* b, int ldb, float* c,
                    int ldc) {
    if (m <= 0 || n <= 0) return;
    if (k <= 0) {
        for (int i = 0; i < m; ++i) std::fill_n(c + size_t(i) * ldc, n, 0.0f);
        return;
    }
    std::vector<float> A(size_t(m) * k), B(size_t(n) * k), Cm(size_t(m) * n);
    for (int i = 0; i < m; ++i) std::copy_n(a + size_t(i) * lda, k, A.data() + size_t(i) * k);
    for (int j = 0; j < n; ++j) std::copy_n(b + size_t(j) * ldb, k, B.data() + size_t(j) * k);
    b200::check(mpic_host_gemm_f32(A.data(), B.data(), uint32_t(m), uint32_t(n), uint32_t(k), Cm.data(),
                                   b200::device()));
    for (int i = 0; i < m; ++i) std::copy_n(Cm.data() + size_t(i) * n, n, c + size_t(i) * ldc);
}
}  // namespace

void gemm_nt(int m, int n, int k, const float* a, int lda, const float* b, int ldb, float* c, int ldc) {
    device_gemm_nt(m, n, k, a, lda, b, ldb, c, ldc);
}

void gemm_nn(int m, int n, int k, const float* a, int lda, const float* b, int ldb, float* c, int ldc) {
    std::vector<float> bt(size_t(n) * std::max(k, 1));  // B[k x n] -> B^T[n x k]
    for (int r = 0; r < k; ++r)
        for (int j = 0; j < n; ++j) bt[size_t(j) * k + r] = b[size_t(r) * ldb + j];
    device_gemm_nt(m, n, k, a, lda, bt.data(), k, c, ldc);
}

void set_compute_threads(int n) { g_threads = n; }

}  // namespace mpic

namespace mpic::b200 {

void check(int rc) {
    if (rc == MPIC_OK) return;
    const std::string msg = mpic_last_error();
    switch (rc) {
        case MPIC_ERR_CONFIG: throw config_error(msg);
        case MPIC_ERR_VALIDATION: throw validation_error(msg);
        case MPIC_ERR_STATE: throw state_error(msg);
        case MPIC_ERR_LINK: throw link_error(msg);
        case MPIC_ERR_CONTRACT: throw contract_error(msg);
        case MPIC_ERR_FORMAT: throw format_error(msg);
        case MPIC_ERR_INTEGRITY: throw integrity_error(msg);
        case MPIC_ERR_IO: throw io_error(msg);
        case MPIC_ERR_NOT_FOUND: throw not_found_error(msg);
        case MPIC_ERR_REQUEST: throw request_error(msg);
        default: throw error("B200 runtime: " + msg);
    }
}

int device() {
    static const int dev = [] {
        const char* e = std::getenv("MPIC_DEVICE");
        return e ? std::atoi(e) : 0;
    }();
    return dev;
}

mpic_dtype compute_dtype() {
    static const mpic_dtype dt = [] {
        const char* e = std::getenv("MPIC_B200_DTYPE");
        return e && std::string(e) == "bf16" ? MPIC_BF16 : MPIC_F32;
    }();
    return dt;
}

mpic_model_config to_c(const ModelConfig& c) {
    mpic_model_config o{};
    o.n_layers = c.n_layers;
    o.n_heads = c.n_heads;
    o.head_dim = c.head_dim;
    o.hidden_dim = c.hidden_dim;
    o.vocab_size = c.vocab_size;
    o.image_token_count = c.image_token_count;
    o.rope_base = c.rope_base;
    o.seed = c.seed;
    return o;
}

DeviceModel::DeviceModel(const Model& m) {
    const mpic_model_config c = to_c(m.config);
    std::vector<const float*> lw;
    lw.reserve(6 * m.layers.size());
    for (const LayerWeights& l : m.layers)
        for (const std::vector<float>* w : {&l.wq, &l.wk, &l.wv, &l.wo, &l.w1, &l.w2}) lw.push_back(w->data());
    check(mpic_model_upload(&c, device(), compute_dtype(), m.embedding.data(), m.lm_head.data(), lw.data(), &h_));
}
DeviceModel::~DeviceModel() { mpic_model_destroy(h_); }

namespace {
struct KvPoolEntry {
    uint32_t L, T, H, D;
    mpic_kv_t h;
};
struct KvPool {
    std::vector<KvPoolEntry> free;
    ~KvPool() {
        for (const KvPoolEntry& e : free) mpic_kv_free(e.h);
    }
};
thread_local KvPool t_kv_pool;
}  // namespace

DeviceKv::DeviceKv(uint32_t layers, uint32_t tokens, uint32_t heads, uint32_t dim) {
    auto& pool = t_kv_pool.free;
    for (auto it = pool.begin(); it != pool.end(); ++it)
        if (it->L == layers && it->T == tokens && it->H == heads && it->D == dim) {
            h_ = it->h;
            pool.erase(it);
            return;
        }
    check(mpic_kv_alloc(layers, tokens, heads, dim, compute_dtype(), device(), &h_));
}
DeviceKv::DeviceKv(const KvTensor& t) : DeviceKv(t.n_layers, t.n_tokens, t.n_heads, t.head_dim) {
    upload(t);
}
DeviceKv::~DeviceKv() {
    uint32_t shape[4];
    mpic_dtype dt;
    auto& pool = t_kv_pool.free;
    if (h_ && mpic_kv_shape(h_, shape, &dt) == MPIC_OK) {
        pool.push_back({shape[0], shape[1], shape[2], shape[3], h_});
        if (pool.size() > 8) {
            mpic_kv_free(pool.front().h);
            pool.erase(pool.begin());
        }
    } else {
        mpic_kv_free(h_);
    }
}
void DeviceKv::upload(const KvTensor& t) {
    if (!t.k.empty()) check(mpic_kv_upload(h_, t.k.data(), t.v.data(), nullptr));
}
void DeviceKv::download(KvTensor& t) const {
    if (!t.k.empty()) check(mpic_kv_download(h_, t.k.data(), t.v.data(), nullptr));
}
void DeviceKv::download_rows(KvTensor& t, std::span<const uint32_t> rows) const {
    if (!t.k.empty() && !rows.empty())
        check(mpic_kv_download_rows(h_, rows.data(), static_cast<uint32_t>(rows.size()), t.k.data(), t.v.data(),
                                    nullptr));
}

Workspace::Workspace(const DeviceModel& m, uint32_t rows, uint32_t ctx) : rows_(std::max(rows, 1u)), ctx_(ctx) {
    check(mpic_workspace_create(m.get(), rows_, ctx, &h_));
}

namespace {
// Identity of a host model's weights for the device-model cache. Models up to
// kFullHashWords weight words (every conformance and test model) hash EVERY word, so any
// in-place edit between calls re-uploads. Larger models (LLaVA width: 6.7 G words, where a
// full pass would cost seconds per call) hash each buffer's address and size plus a strided
// sample of its words; callers that edit such a model in place must build a new Model (the
// reference treats Model as immutable after build_model, model.h:22-30).
constexpr size_t kFullHashWords = size_t(64) << 20;  // 256 MB of fp32 weights

size_t weight_words(const Model& m) {
    size_t n = m.embedding.size() + m.lm_head.size();
    for (const LayerWeights& l : m.layers)
        n += l.wq.size() + l.wk.size() + l.wv.size() + l.wo.size() + l.w1.size() + l.w2.size();
    return n;
}

uint64_t weight_hash(const Model& m) {
    const bool full = weight_words(m) <= kFullHashWords;
    uint64_t acc = 0x9e3779b97f4a7c15ull ^ m.config.fingerprint();
    auto mix = [&](uint64_t v) { acc = (acc ^ v) * 0x100000001b3ull; };
    auto feed = [&](const std::vector<float>& w) {
        const auto* p = reinterpret_cast<const uint32_t*>(w.data());
        const size_t n = w.size();
        mix(reinterpret_cast<uintptr_t>(p));
        mix(n);
        if (full) {
            // four independent multiply-xor lanes over 64-bit words (~10 GB/s)
            uint64_t a[4] = {1, 2, 3, 4};
            const auto* q = reinterpret_cast<const uint64_t*>(p);
            const size_t n64 = n / 2;
            size_t i = 0;
            for (; i + 4 <= n64; i += 4)
                for (int j = 0; j < 4; ++j) a[j] = (a[j] ^ q[i + j]) * 0x9fb21c651e98df25ull;
            for (; i < n64; ++i) a[0] = (a[0] ^ q[i]) * 0x9fb21c651e98df25ull;
            if (n & 1) a[1] = (a[1] ^ p[n - 1]) * 0x9fb21c651e98df25ull;
            for (int j = 0; j < 4; ++j) mix(a[j] ^ (a[j] >> 29));
        } else {
            const size_t step = std::max<size_t>(1, n / 61);
            for (size_t i = 0; i < n; i += step) mix(p[i]);
            if (n) mix(p[n - 1]);
        }
    };
    feed(m.embedding);
    feed(m.lm_head);
    for (const LayerWeights& l : m.layers)
        for (const std::vector<float>* w : {&l.wq, &l.wk, &l.wv, &l.wo, &l.w1, &l.w2}) feed(*w);
    return acc;
}

struct ModelCacheEntry {
    const Model* addr;
    uint64_t hash;
    std::shared_ptr<DeviceModel> dev;
};
std::mutex g_model_cache_mu;
std::vector<ModelCacheEntry> g_model_cache;  // most recent last, at most 4 entries

struct WsCacheEntry {
    std::shared_ptr<DeviceModel> model;
    std::unique_ptr<Workspace> ws;
};
thread_local std::vector<WsCacheEntry> t_ws_cache;
}  // namespace

std::shared_ptr<DeviceModel> device_model_for(const Model& m) {
    const uint64_t h = weight_hash(m);
    std::lock_guard<std::mutex> lk(g_model_cache_mu);
    for (auto it = g_model_cache.begin(); it != g_model_cache.end(); ++it)
        if (it->addr == &m && it->hash == h) {
            ModelCacheEntry e = *it;
            g_model_cache.erase(it);
            g_model_cache.push_back(e);
            return e.dev;
        }
    auto dev = std::make_shared<DeviceModel>(m);
    g_model_cache.push_back({&m, h, dev});
    if (g_model_cache.size() > 4) g_model_cache.erase(g_model_cache.begin());
    return dev;
}

Workspace& workspace_for(const std::shared_ptr<DeviceModel>& m, uint32_t rows, uint32_t ctx) {
    for (auto it = t_ws_cache.begin(); it != t_ws_cache.end(); ++it)
        if (it->model == m) {
            if (it->ws->rows() < rows || it->ws->ctx() < ctx)
                it->ws = std::make_unique<Workspace>(*m, std::max(rows, it->ws->rows()), std::max(ctx, it->ws->ctx()));
            return *it->ws;
        }
    // drop workspaces of models that left the model cache
    t_ws_cache.erase(std::remove_if(t_ws_cache.begin(), t_ws_cache.end(),
                                    [](const WsCacheEntry& e) { return e.model.use_count() <= 1; }),
                     t_ws_cache.end());
    t_ws_cache.push_back({m, std::make_unique<Workspace>(*m, rows, ctx)});
    return *t_ws_cache.back().ws;
}
Workspace::~Workspace() { mpic_workspace_destroy(h_); }

}  // namespace mpic::b200
