// C ABI of the MPIC B200 path (include/mpic_b200.h): handles, the per-layer launch
// sequence of the selective recompute, and the assembly entry points.
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>
#include <zlib.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cerrno>
#include <cmath>
#include <condition_variable>
#include <cstring>
#include <memory>
#include <thread>
#include <mutex>
#include <functional>
#include <mutex>
#include <string>
#include <type_traits>
#include <vector>

#include "common.cuh"
#include "kernels.h"

namespace mpicb {
namespace {
thread_local std::string g_last_error;
thread_local uint32_t g_launches = 0;
}  // namespace
void note_launch(uint32_t n) { g_launches += n; }
void set_last_error(const std::string& m) { g_last_error = m; }
bool pdl_enabled() {
    static const bool on = [] {
        const char* e = getenv("MPIC_PDL");
        return !e || atoi(e) != 0;
    }();
    return on;
}

// MPIC_ATTN_FUSED_COMBINE=1 (diagnostics): the split that completes a (tile, head) merges the
// partials inside the attention kernel instead of attn_combine_kernel. Measured slower at
// config C (attention 2.85 -> 4.32 ms per request): a merge is a latency-bound read of up to
// 16 x 64 KB by one warpgroup, on the critical path of whichever CTA finishes a job last.
static bool fused_combine() {
    static const bool on = [] {
        const char* e = getenv("MPIC_ATTN_FUSED_COMBINE");
        return e && atoi(e) != 0;
    }();
    return on;
}

// Scheduling priority of the request's hot kernels (GEMMs, attention): above the default
// priority of the side-stream assembly, so assembly CTAs only fill SMs the hot path leaves
// idle. MPIC_PRIO=0 (diagnostics) launches everything at the default priority.
int hot_priority() {
    static const int prio = [] {
        const char* e = getenv("MPIC_PRIO");
        if (e && atoi(e) == 0) return 0;
        int least = 0, greatest = 0;
        if (cudaDeviceGetStreamPriorityRange(&least, &greatest) != cudaSuccess) return 0;
        return greatest;
    }();
    return prio;
}

// ---- per-phase device timing (CUDA events on the launching stream) ------------------
// Enabled by mpic_profile_enable(1); each phase of a forward/assembly records a start and
// stop event around its launches; mpic_profile_collect() synchronizes and sums them.
namespace {
struct ProfRec {
    int cls;
    cudaEvent_t a, b;
};
std::mutex g_prof_mu;
bool g_prof_on = false;
std::vector<ProfRec> g_prof_recs;
std::vector<cudaEvent_t> g_prof_pool;

cudaEvent_t prof_event() {
    if (!g_prof_pool.empty()) {
        cudaEvent_t e = g_prof_pool.back();
        g_prof_pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    MPIC_CUDA(cudaEventCreate(&e));
    return e;
}
}  // namespace

struct ProfScope {
    cudaStream_t s;
    int cls;
    cudaEvent_t a = nullptr;
    ProfScope(cudaStream_t st, int c) : s(st), cls(c) {
        if (!g_prof_on) return;
        std::lock_guard<std::mutex> lk(g_prof_mu);
        a = prof_event();
        cudaEventRecord(a, s);
    }
    ~ProfScope() {
        if (!a) return;
        std::lock_guard<std::mutex> lk(g_prof_mu);
        cudaEvent_t b = prof_event();
        cudaEventRecord(b, s);
        g_prof_recs.push_back({cls, a, b});
    }
};
}  // namespace mpicb

using namespace mpicb;

struct mpic_model_s {
    mpic_model_config cfg{};
    int device = 0;
    mpic_dtype dtype = MPIC_F32;
    float* emb = nullptr;      // [V][h] fp32 (gathered, never multiplied)
    void* lm_head = nullptr;   // [V][h] dtype
    std::vector<void*> wqkv;   // per layer [3h][h]: wq | wk | wv rows
    std::vector<void*> wo;     // [h][h]
    std::vector<void*> w1;     // [4h][h]
    std::vector<void*> w2;     // [h][4h]
    double* inv_freq = nullptr;  // [D/2]
    float2* rope = nullptr;      // [rope_cap][D/2]
    uint32_t rope_cap = 0;
    std::vector<float2*> retired;  // old tables kept alive (other streams may read them)
    std::mutex mu;
    // head-parallel slice (mpic_model_create_heads): attention weights of heads
    // [head0, head0 + n_local_heads) only; 0 local heads = the whole model
    uint32_t head0 = 0, n_local_heads = 0;
    // fp32 mode on the tensor cores (3xTF32): the tf32 hi / lo split of every projection
    // weight, keyed by the weight's pointer (weights are immutable after creation)
    std::unordered_map<const void*, std::pair<float*, float*>> x3w;
};

struct mpic_kv_s {
    uint32_t L = 0, T = 0, H = 0, D = 0;
    mpic_dtype dtype = MPIC_F32;
    int device = 0;
    void* k = nullptr;
    void* v = nullptr;
    size_t elems() const { return (size_t)L * T * H * D; }
};

// Everything that fixes the launch sequence of a device-resident request: same signature
// => same kernels, grids and tensor maps; only the staged inputs differ.
// The graph holds raw device/pinned pointers: the linked cache's K/V planes (not the handle,
// whose address a later allocation may reuse), the model's RoPE table, and the workspace
// buffers, whose reallocations bump `ws_gen`.
struct GraphSig {
    const void* model = nullptr;
    const void* linked_k = nullptr;
    const void* linked_v = nullptr;
    const void* rope = nullptr;
    uint64_t ws_gen = 0;
    uint32_t n = 0, m = 0, n_img = 0, n_tables = 0, n_units = 0, n_comb = 0;
    int reposition = 0, src_dtype = 0;
    bool link = false;
    bool operator==(const GraphSig& o) const {
        return model == o.model && linked_k == o.linked_k && linked_v == o.linked_v && rope == o.rope &&
               ws_gen == o.ws_gen && n == o.n && m == o.m && n_img == o.n_img && n_tables == o.n_tables &&
               n_units == o.n_units && n_comb == o.n_comb && reposition == o.reposition &&
               src_dtype == o.src_dtype && link == o.link;
    }
};

struct mpic_workspace_s {
    mpic_model_t model = nullptr;
    uint32_t max_rows = 0, max_ctx = 0, m_pad = 0;
    int32_t* d_ids = nullptr;
    uint32_t* d_rows = nullptr;
    uint32_t* d_pos = nullptr;
    uint32_t* d_start = nullptr;        // batched requests: first cache row of each row's request
    float* x = nullptr;                 // residual stream fp32 [m_pad][h]
    float2* rope_tok = nullptr;         // (cos, sin) of each row's position [m_pad][D/2]
    __nv_bfloat16* xb = nullptr;        // bf16 copy of x (GEMM A operand, bf16 mode)
    void* q = nullptr;                  // [m_pad][h] dtype
    void* attn = nullptr;               // [m_pad][h] dtype
    void* ffn = nullptr;                // [m_pad][4h] dtype
    float* d_logits = nullptr;          // [V]
    float* partial = nullptr;           // split-K partials [8][m_pad][h]
    float* x3buf = nullptr;             // fp32 mode, 3xTF32: tf32 hi / lo split of a GEMM's A [2][m_pad][4h]
    size_t partial_cap = 0;
    int32_t* h_ids = nullptr;           // pinned staging
    uint32_t* h_rows = nullptr;
    uint32_t* h_pos = nullptr;
    uint32_t* h_start = nullptr;
    float* h_logits = nullptr;
    // loader lane (mpic_request_prefill_host): side stream, 2-slot HBM staging ring
    cudaStream_t copy_stream = nullptr;
    cudaEvent_t ev_ready[2] = {nullptr, nullptr};
    cudaEvent_t ev_free[2] = {nullptr, nullptr};
    void* stage[2] = {nullptr, nullptr};
    size_t stage_cap = 0;
    // disk loader (mpic_request_prefill_files): pinned ring of layer slots
    void* pin[3] = {nullptr, nullptr, nullptr};
    cudaEvent_t ev_pin[3] = {nullptr, nullptr, nullptr};
    size_t pin_cap = 0;
    // tcgen05 attention plan (per request) and split partials
    AttnUnit* d_units = nullptr;
    AttnCombine* d_comb = nullptr;
    uint32_t* d_comb_cnt = nullptr;  // fused combine: per job, splits finished (self-resetting, zeroed once)
    size_t units_cap = 0, comb_cap = 0, comb_cnt_cap = 0;
    float* part_o = nullptr;
    float2* part_ml = nullptr;
    size_t slots_cap = 0;
    void* h_plan = nullptr;  // pinned staging for the plan
    size_t h_plan_cap = 0;
    uint32_t n_units = 0, n_unit_entries = 0, n_comb = 0;
    cudaEvent_t ev_plan = nullptr;
    // assembly descriptors (AsmChunk table + rerotation tables), pinned staging + device copy
    void* h_asm = nullptr;
    void* d_asm = nullptr;
    size_t asm_cap = 0;
    // CUDA-graph replay of a device-resident request (mpic_request_prefill): the request
    // whose shape matches the previous one is captured once, later ones replay it
    bool graphs = true;
    uint64_t gen = 0;  // bumped whenever a buffer a recorded graph may reference is reallocated
    GraphSig last_sig{}, graph_sig{};
    cudaGraphExec_t graph = nullptr;
    uint32_t graph_kernels = 0;
    uint32_t hp_m = 0, hp_n = 0;  // head-parallel request in flight (mpic_hp_prepare)
    // per-layer assembly overlapped with the layer loop (mpic_request_prefill)
    cudaStream_t asm_stream = nullptr;
    cudaEvent_t ev_asm_in = nullptr;
    std::vector<cudaEvent_t> ev_asm;
    // compute lane of the loader paths (prepare's compute lane, transfer.cpp:119-127): chunks
    // that are missing or fail to load are prefilled on their own stream and workspace
    mpic_workspace_s* aux = nullptr;
    cudaStream_t miss_stream = nullptr;
    // the compute lane's chunk buffers, kept across requests (allocating and freeing ~1 GB
    // chunk tensors per request cost more than computing them)
    struct MissBuf {
        void* k = nullptr;
        void* v = nullptr;
        int32_t* d_ids = nullptr;
        uint32_t* d_rows = nullptr;
        size_t bytes = 0;
        uint32_t rows = 0;
        std::vector<cudaEvent_t> ev;
    };
    std::vector<MissBuf> miss_pool;
    // head-parallel request inside the library (mpic_hp_request): Wo partials [m_pad][h] and
    // this rank's reduced rows [mr][h] (fp32), and the captured layer loop
    float* hp_partial = nullptr;
    float* hp_reduced = nullptr;
    size_t hp_partial_cap = 0, hp_reduced_cap = 0;
    cudaGraphExec_t hp_graph = nullptr;
    uint64_t hp_graph_key = 0, hp_last_key = 0;
    uint32_t hp_graph_kernels = 0;
};

#define API_BEGIN \
    try {         \
        g_launches = 0;
#define API_END                                   \
    return MPIC_OK;                               \
    }                                             \
    catch (const mpicb::Error& e) {               \
        mpicb::g_last_error = e.what();           \
        return e.code;                            \
    }                                             \
    catch (const std::exception& e) {             \
        mpicb::g_last_error = e.what();           \
        return MPIC_ERR_CUDA;                     \
    }

namespace {

void set_device(int dev) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0)
        throw Error(MPIC_ERR_NO_DEVICE, "no CUDA device: the MPIC B200 path has no CPU fallback");
    MPIC_REQUIRE(dev >= 0 && dev < n, MPIC_ERR_VALIDATION, "device index out of range");
    MPIC_CUDA(cudaSetDevice(dev));
    cudaDeviceProp p;
    MPIC_CUDA(cudaGetDeviceProperties(&p, dev));
    if (p.major != 10)
        throw Error(MPIC_ERR_NO_DEVICE, std::string("device ") + p.name +
                                            " is not sm_100 (this library is built for sm_100a only)");
}

void validate_cfg(const mpic_model_config* c) {
    MPIC_REQUIRE(c, MPIC_ERR_VALIDATION, "null config");
    // ModelConfig::validate (proj/src/config.cpp:12-28)
    MPIC_REQUIRE(c->n_layers && c->n_heads && c->head_dim && c->hidden_dim, MPIC_ERR_CONFIG,
                 "model dimensions must be positive");
    MPIC_REQUIRE(c->hidden_dim == c->n_heads * c->head_dim, MPIC_ERR_CONFIG,
                 "hidden_dim must equal n_heads * head_dim");
    MPIC_REQUIRE(c->vocab_size >= 2, MPIC_ERR_CONFIG, "vocab_size must be at least 2");
    MPIC_REQUIRE(c->image_token_count > 0, MPIC_ERR_CONFIG, "image_token_count must be positive");
    MPIC_REQUIRE(c->rope_base > 0.0f, MPIC_ERR_CONFIG, "rope_base must be positive");
}

void validate_device_cfg(const mpic_model_config* c) {
    // Limits of this implementation (documented in DESIGN.md).
    MPIC_REQUIRE(c->head_dim % 2 == 0, MPIC_ERR_CONFIG, "head_dim must be even on the B200 path");
    MPIC_REQUIRE(c->head_dim <= 256, MPIC_ERR_CONFIG, "head_dim must be <= 256 on the B200 path");
}

template <typename T>
T* dmalloc(size_t n) {
    void* p = nullptr;
    if (n == 0) n = 1;
    MPIC_CUDA(cudaMalloc(&p, n * sizeof(T)));
    return static_cast<T*>(p);
}

size_t esz(mpic_dtype d) { return d == MPIC_BF16 ? 2 : 4; }

void free_model(mpic_model_t m) {
    if (!m) return;
    cudaSetDevice(m->device);
    cudaFree(m->emb);
    cudaFree(m->lm_head);
    for (auto* p : m->wqkv) cudaFree(p);
    for (auto* p : m->wo) cudaFree(p);
    for (auto* p : m->w1) cudaFree(p);
    for (auto* p : m->w2) cudaFree(p);
    cudaFree(m->inv_freq);
    cudaFree(m->rope);
    for (auto* p : m->retired) cudaFree(p);
    for (auto& kv : m->x3w) {
        cudaFree(kv.second.first);
        cudaFree(kv.second.second);
    }
    delete m;
}

// fp32 projections on the tensor cores (3xTF32, tc_pgemm.cu) unless MPIC_F32_GEMM=simt
// selects the SIMT FFMA GEMM (simt.cu).
bool f32_tensor_gemm() {
    static const bool on = [] {
        const char* e = getenv("MPIC_F32_GEMM");
        return !(e && std::string(e) == "simt");
    }();
    return on;
}

// Split every projection weight of an fp32 model whose shape the 3xTF32 GEMM takes.
void prepare_x3(mpic_model_t m, cudaStream_t s) {
    if (m->dtype != MPIC_F32 || !f32_tensor_gemm() || m->n_local_heads) return;
    const size_t h = m->cfg.hidden_dim;
    auto split = [&](const void* w, size_t N, size_t K) {
        if (!pgemm_x3_supported(1, (uint32_t)N, (uint32_t)K)) return;
        float* hi = dmalloc<float>(N * K);
        float* lo = dmalloc<float>(N * K);
        launch_tf32_split(static_cast<const float*>(w), hi, lo, N * K, s);
        m->x3w[w] = {hi, lo};
    };
    for (size_t l = 0; l < m->cfg.n_layers; ++l) {
        split(m->wqkv[l], 3 * h, h);
        split(m->wo[l], h, h);
        split(m->w1[l], 4 * h, h);
        split(m->w2[l], h, 4 * h);
    }
}

void alloc_model(mpic_model_t m) {
    const size_t h = m->cfg.hidden_dim, V = m->cfg.vocab_size, L = m->cfg.n_layers;
    const size_t e = esz(m->dtype);
    m->emb = dmalloc<float>(V * h);
    MPIC_CUDA(cudaMalloc(&m->lm_head, V * h * e));
    for (size_t l = 0; l < L; ++l) {
        void* p;
        MPIC_CUDA(cudaMalloc(&p, 3 * h * h * e));
        m->wqkv.push_back(p);
        MPIC_CUDA(cudaMalloc(&p, h * h * e));
        m->wo.push_back(p);
        MPIC_CUDA(cudaMalloc(&p, 4 * h * h * e));
        m->w1.push_back(p);
        MPIC_CUDA(cudaMalloc(&p, 4 * h * h * e));
        m->w2.push_back(p);
    }
    const uint32_t D = m->cfg.head_dim;
    std::vector<double> inv(D / 2);
    for (uint32_t i = 0; i + 1 < D; i += 2)  // model.cpp:51-53
        inv[i / 2] = std::pow(static_cast<double>(m->cfg.rope_base), -static_cast<double>(i) / D);
    m->inv_freq = dmalloc<double>(D / 2);
    MPIC_CUDA(cudaMemcpy(m->inv_freq, inv.data(), inv.size() * sizeof(double), cudaMemcpyHostToDevice));
}

// Pointer to weight `which` (0 emb, 1 lm_head, 2..7 wq wk wv wo w1 w2) and its size.
void* weight_ptr(mpic_model_t m, int which, uint32_t layer, size_t* count) {
    const size_t h = m->cfg.hidden_dim, V = m->cfg.vocab_size;
    const size_t e = esz(m->dtype);
    MPIC_REQUIRE(which >= 0 && which <= 7, MPIC_ERR_VALIDATION, "bad weight index");
    MPIC_REQUIRE(which < 2 || layer < m->cfg.n_layers, MPIC_ERR_VALIDATION, "layer out of range");
    switch (which) {
        case 0: *count = V * h; return m->emb;
        case 1: *count = V * h; return m->lm_head;
        case 2: *count = h * h; return m->wqkv[layer];
        case 3: *count = h * h; return (char*)m->wqkv[layer] + h * h * e;
        case 4: *count = h * h; return (char*)m->wqkv[layer] + 2 * h * h * e;
        case 5: *count = h * h; return m->wo[layer];
        case 6: *count = 4 * h * h; return m->w1[layer];
        default: *count = 4 * h * h; return m->w2[layer];
    }
}

// Grow the cached RoPE (cos, sin) table to cover positions [0, need).
void ensure_rope(mpic_model_t m, uint32_t need, cudaStream_t s) {
    std::lock_guard<std::mutex> lk(m->mu);
    if (need <= m->rope_cap) return;
    uint32_t cap = 4096;
    while (cap < need) cap *= 2;
    const uint32_t half = m->cfg.head_dim / 2;
    float2* t = dmalloc<float2>((size_t)cap * half);
    launch_rope_table(m->inv_freq, half, 0, cap, t, s);
    MPIC_CUDA(cudaStreamSynchronize(s));
    if (m->rope) m->retired.push_back(m->rope);
    m->rope = t;
    m->rope_cap = cap;
}

// Upload n host fp32 values into a device buffer of dtype dt (cast on device).
void upload_cast(void* dst, mpic_dtype dt, const float* src, size_t n, cudaStream_t s) {
    if (dt == MPIC_F32) {
        MPIC_CUDA(cudaMemcpyAsync(dst, src, n * 4, cudaMemcpyHostToDevice, s));
        MPIC_CUDA(cudaStreamSynchronize(s));
        return;
    }
    const size_t chunk = std::min<size_t>(n, (size_t)64 << 20);
    float* tmp = dmalloc<float>(chunk);
    for (size_t off = 0; off < n; off += chunk) {
        const size_t c = std::min(chunk, n - off);
        MPIC_CUDA(cudaMemcpyAsync(tmp, src + off, c * 4, cudaMemcpyHostToDevice, s));
        launch_f32_to_bf16(tmp, static_cast<__nv_bfloat16*>(dst) + off, c, s);
    }
    MPIC_CUDA(cudaStreamSynchronize(s));
    cudaFree(tmp);
}

void download_cast(float* dst, const void* src, mpic_dtype dt, size_t n, cudaStream_t s) {
    if (dt == MPIC_F32) {
        MPIC_CUDA(cudaMemcpyAsync(dst, src, n * 4, cudaMemcpyDeviceToHost, s));
        MPIC_CUDA(cudaStreamSynchronize(s));
        return;
    }
    const size_t chunk = std::min<size_t>(n, (size_t)64 << 20);
    float* tmp = dmalloc<float>(chunk);
    for (size_t off = 0; off < n; off += chunk) {
        const size_t c = std::min(chunk, n - off);
        launch_bf16_to_f32(static_cast<const __nv_bfloat16*>(src) + off, tmp, c, s);
        MPIC_CUDA(cudaMemcpyAsync(dst + off, tmp, c * 4, cudaMemcpyDeviceToHost, s));
    }
    MPIC_CUDA(cudaStreamSynchronize(s));
    cudaFree(tmp);
}

// One projection GEMM with its fused epilogue: tcgen05 for bf16; for fp32, 3xTF32 tcgen05
// when the weight has its split and the caller passes split scratch for A (x3buf: 2 x M x K
// floats), else SIMT FFMA.
void run_gemm(mpic_model_t md, const void* A, const void* W, uint32_t M, uint32_t N, uint32_t K,
              const EpiParams& ep, cudaStream_t s, float* x3buf = nullptr) {
    if (md->dtype == MPIC_BF16) {
        if (tc_gemm_supported(M, N, K) && (ep.mode != EPI_QKV || md->cfg.head_dim % 32 == 0)) {
            launch_gemm_tc(static_cast<const __nv_bfloat16*>(A), K,
                           static_cast<const __nv_bfloat16*>(W), M, N, K, ep, s);
            return;
        }
        EpiParams e2 = ep;
        e2.split_k = 1;
        launch_gemm_simt(A, MPIC_BF16, K, W, MPIC_BF16, M, N, K, e2, MPIC_BF16, s);
        return;
    }
    if (x3buf && pgemm_x3_supported(M, N, K)) {
        const auto it = md->x3w.find(W);
        if (it != md->x3w.end()) {
            float* a_hi = x3buf;
            float* a_lo = x3buf + (size_t)M * K;
            launch_tf32_split(static_cast<const float*>(A), a_hi, a_lo, (size_t)M * K, s);
            launch_pgemm_x3(a_hi, a_lo, it->second.first, it->second.second, M, N, K, ep, s);
            return;
        }
    }
    launch_gemm_simt(A, MPIC_F32, K, W, MPIC_F32, M, N, K, ep, MPIC_F32, s);
}

bool use_tc_attention(mpic_model_t md) {
    return md->dtype == MPIC_BF16 && md->cfg.head_dim == 128;
}

bool attn_link_enabled() {
    static const bool on = [] {
        const char* e = getenv("MPIC_ATTN_LINK");  // diagnostics: 0 = assemble every block up front
        return !e || atoi(e) != 0;
    }();
    return on;
}

// Blocks of 128 cache rows that attention can read straight from a cached chunk (AttnLink):
// inside one chunk's destination range and holding no recomputed row. Returns false when no
// block qualifies. blk / skip are per block (kernels.h AttnLink; skip = not assembled).
bool plan_attn_link(const std::vector<mpic_chunk_ref>& refs, const uint32_t* sel, uint32_t m, uint32_t n,
                    std::vector<uint32_t>& blk, std::vector<uint16_t>& wtile, std::vector<uint8_t>& skip) {
    const uint32_t nblk = (n + 127) / 128;
    blk.assign(nblk, kLinkedBlock);
    // writer tile: the lowest query tile whose key range reaches the block (the attention
    // plan's per-tile range is [0, rows[last row of the tile] / 128])
    wtile.assign(nblk, 0);
    {
        uint32_t t = 0;
        for (uint32_t b = 0; b < nblk; ++b) {
            while (t + 1 < (m + 127) / 128 && sel[attn_tile_last_row(t, m)] / 128 < b) ++t;
            wtile[b] = (uint16_t)t;
        }
    }
    skip.assign(nblk, 0);
    std::vector<uint8_t> rec(n, 0);
    for (uint32_t i = 0; i < m; ++i)
        if (sel[i] < n) rec[sel[i]] = 1;
    bool any = false;
    for (uint32_t b = 0; b * 128 + 128 <= n; ++b) {
        const uint32_t a0 = b * 128;
        for (uint32_t c = 0; c < refs.size(); ++c) {
            const mpic_chunk_ref& ref = refs[c];
            if (a0 < ref.dst_row0 || a0 + 128 > ref.dst_row0 + ref.rows) continue;
            bool recomputed = false;
            for (uint32_t k = a0; k < a0 + 128 && !recomputed; ++k) recomputed = rec[k] != 0;
            const uint32_t src = ref.src_row0 + (a0 - ref.dst_row0);
            if (!recomputed && src < (1u << 24)) {
                blk[b] = (c << 24) | src;
                skip[b] = 1;
                any = true;
            }
            break;
        }
    }
    return any;
}

// Build the attention work plan from host rows (or, without them, a conservative plan in
// which every query may see keys up to max_pos), grow the workspace buffers it needs and
// stage it in pinned memory. Host-only: nothing is enqueued, so it may run before a
// stream capture. enqueue_attn_plan() then copies it to the device on the stream.
void prepare_attn_plan(mpic_workspace_t ws, const uint32_t* h_rows, uint32_t m, uint32_t max_pos, uint32_t H,
                       const uint32_t* h_starts = nullptr) {
    std::vector<uint32_t> conservative;
    if (!h_rows) {
        conservative.assign(m, max_pos);
        h_rows = conservative.data();
    }
    const AttnPlan plan = plan_attention(h_rows, m, H, h_starts);
    auto grow = [&](auto*& ptr, size_t& cap, size_t need, size_t elt) {
        if (cap >= need) return;
        ++ws->gen;
        MPIC_CUDA(cudaDeviceSynchronize());
        cudaFree(ptr);
        ptr = nullptr;
        MPIC_CUDA(cudaMalloc((void**)&ptr, std::max<size_t>(need, 1) * elt));
        cap = need;
    };
    grow(ws->d_units, ws->units_cap, plan.units.size(), sizeof(AttnUnit));
    grow(ws->d_comb, ws->comb_cap, plan.combine.size(), sizeof(AttnCombine));
    if (ws->comb_cnt_cap < plan.combine.size()) {  // the kernel leaves every counter at 0
        ++ws->gen;
        MPIC_CUDA(cudaDeviceSynchronize());
        cudaFree(ws->d_comb_cnt);
        MPIC_CUDA(cudaMalloc(&ws->d_comb_cnt, plan.combine.size() * sizeof(uint32_t)));
        MPIC_CUDA(cudaMemset(ws->d_comb_cnt, 0, plan.combine.size() * sizeof(uint32_t)));
        ws->comb_cnt_cap = plan.combine.size();
    }
    if (ws->slots_cap < plan.slots) {
        ++ws->gen;
        MPIC_CUDA(cudaDeviceSynchronize());
        cudaFree(ws->part_o);
        cudaFree(ws->part_ml);
        MPIC_CUDA(cudaMalloc(&ws->part_o, (size_t)plan.slots * 128 * 128 * sizeof(float)));
        MPIC_CUDA(cudaMalloc(&ws->part_ml, (size_t)plan.slots * 128 * sizeof(float2)));
        ws->slots_cap = plan.slots;
    }
    const size_t bu = plan.units.size() * sizeof(AttnUnit);
    const size_t bc = plan.combine.size() * sizeof(AttnCombine);
    // the previous request's copy out of the pinned staging must have landed
    if (ws->ev_plan) MPIC_CUDA(cudaEventSynchronize(ws->ev_plan));
    if (ws->h_plan_cap < bu + bc) {
        ++ws->gen;
        cudaFreeHost(ws->h_plan);
        MPIC_CUDA(cudaMallocHost(&ws->h_plan, bu + bc));
        ws->h_plan_cap = bu + bc;
    }
    std::memcpy(ws->h_plan, plan.units.data(), bu);
    std::memcpy((char*)ws->h_plan + bu, plan.combine.data(), bc);
    ws->n_units = plan.items;  // work items; the per-CTA offsets follow them (AttnPlan)
    ws->n_unit_entries = (uint32_t)plan.units.size();
    ws->n_comb = (uint32_t)plan.combine.size();
}

void enqueue_attn_plan(mpic_workspace_t ws, cudaStream_t s) {
    const size_t bu = ws->n_unit_entries * sizeof(AttnUnit), bc = ws->n_comb * sizeof(AttnCombine);
    if (bu) MPIC_CUDA(cudaMemcpyAsync(ws->d_units, ws->h_plan, bu, cudaMemcpyHostToDevice, s));
    if (bc) MPIC_CUDA(cudaMemcpyAsync(ws->d_comb, (char*)ws->h_plan + bu, bc, cudaMemcpyHostToDevice, s));
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    MPIC_CUDA(cudaStreamIsCapturing(s, &cs));
    if (cs != cudaStreamCaptureStatusNone) return;  // graph requests end in a stream sync
    if (!ws->ev_plan) MPIC_CUDA(cudaEventCreateWithFlags(&ws->ev_plan, cudaEventDisableTiming));
    MPIC_CUDA(cudaEventRecord(ws->ev_plan, s));
}

void ensure_asm_stream(mpic_workspace_t ws, uint32_t layers) {
    if (!ws->asm_stream) {
        MPIC_CUDA(cudaStreamCreateWithFlags(&ws->asm_stream, cudaStreamNonBlocking));
        MPIC_CUDA(cudaEventCreateWithFlags(&ws->ev_asm_in, cudaEventDisableTiming));
    }
    while (ws->ev_asm.size() < layers) {
        cudaEvent_t e;
        MPIC_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        ws->ev_asm.push_back(e);
    }
}

// selective_core / extend_rows on the device (linker.cpp:35-135, model.cpp:211-330).
void forward_rows(mpic_model_t md, mpic_workspace_t ws, const int32_t* d_ids,
                  const uint32_t* d_rows, const uint32_t* d_pos, uint32_t m, uint32_t max_pos,
                  mpic_kv_t kv, float* d_logits, cudaStream_t s,
                  const std::function<void(uint32_t)>& before_layer = {},
                  const uint32_t* h_rows = nullptr, float* d_capture = nullptr, bool plan_ready = false,
                  const AttnLink* d_link = nullptr, const uint32_t* d_starts = nullptr,
                  const std::vector<uint32_t>* logit_rows = nullptr) {
    const mpic_model_config& c = md->cfg;
    const uint32_t h = c.hidden_dim, H = c.n_heads, D = c.head_dim;
    MPIC_REQUIRE(m > 0, MPIC_ERR_VALIDATION, "no tokens to prefill");
    MPIC_REQUIRE(m <= ws->max_rows, MPIC_ERR_VALIDATION, "more rows than the workspace holds");
    MPIC_REQUIRE(kv->L == c.n_layers && kv->H == H && kv->D == D, MPIC_ERR_VALIDATION,
                 "cache shape does not match model");
    MPIC_REQUIRE(kv->dtype == md->dtype, MPIC_ERR_VALIDATION, "cache dtype does not match model");
    ensure_rope(md, max_pos + 1, s);
    const bool bf = md->dtype == MPIC_BF16;
    const size_t e = esz(md->dtype);
    const size_t plane = (size_t)kv->T * h * e;

    {
        ProfScope ps(s, MPIC_PHASE_EMBED);
        launch_embed(md->emb, d_ids, m, h, ws->x, bf ? ws->xb : nullptr, s);
    }
    if (bf) launch_rope_gather(md->rope, d_pos, m, D / 2, ws->rope_tok, s);
    const bool tc_attn = use_tc_attention(md);
    if (tc_attn) {
        if (!plan_ready) prepare_attn_plan(ws, h_rows, m, max_pos, H);
        enqueue_attn_plan(ws, s);
    }
    for (uint32_t l = 0; l < c.n_layers; ++l) {
        void* kl = (char*)kv->k + l * plane;
        void* vl = (char*)kv->v + l * plane;
        if (before_layer) before_layer(l);
        EpiParams qkv;
        qkv.mode = EPI_QKV;
        qkv.q = ws->q;
        qkv.kv_k = kl;
        qkv.kv_v = vl;
        qkv.kv_rows = d_rows;
        qkv.rope_pos = d_pos;
        qkv.rope = md->rope;
        qkv.rope_tok = bf ? ws->rope_tok : nullptr;
        qkv.hidden = h;
        qkv.head_dim = D;
        {
            ProfScope ps(s, MPIC_PHASE_QKV);
            run_gemm(md, bf ? (const void*)ws->xb : (const void*)ws->x, md->wqkv[l], m, 3 * h, h, qkv, s, ws->x3buf);
        }
        {
            ProfScope ps(s, MPIC_PHASE_ATTN);
            if (d_capture)
                launch_attn_simt(ws->q, kl, vl, md->dtype, d_rows, m, H, D, ws->attn, s,
                                 d_capture + (size_t)l * H * kv->T * kv->T, kv->T);
            else if (tc_attn)
                launch_attn_tc(static_cast<const __nv_bfloat16*>(ws->q), static_cast<const __nv_bfloat16*>(kl),
                               static_cast<const __nv_bfloat16*>(vl), kv->T, d_rows, m, H, ws->d_units,
                               ws->n_units, ws->d_comb, ws->n_comb, ws->part_o, ws->part_ml,
                               static_cast<__nv_bfloat16*>(ws->attn), s, d_link, l, d_starts,
                               fused_combine() ? ws->d_comb_cnt : nullptr);
            else  // fp32: the 3xTF32 GEMMs' split scratch is idle during attention
                launch_attn_simt(ws->q, kl, vl, md->dtype, d_rows, m, H, D, ws->attn, s, nullptr, 0, ws->x3buf,
                                 ws->x3buf ? (size_t)8 * ws->m_pad * h : 0);
        }

        EpiParams res;
        res.mode = EPI_RESID;
        res.x = ws->x;
        res.ldx = h;
        if (bf) {  // residual add also emits the bf16 operand of the next GEMM
            res.xb = ws->xb;
            res.partial = ws->partial;
            res.partial_cap = ws->partial_cap;
        }
        {
            ProfScope ps(s, MPIC_PHASE_WO);
            run_gemm(md, ws->attn, md->wo[l], m, h, h, res, s, ws->x3buf);
        }

        EpiParams gl;
        gl.mode = EPI_GELU;
        gl.out = ws->ffn;
        gl.ldo = 4 * h;
        {
            ProfScope ps(s, MPIC_PHASE_W1);
            run_gemm(md, bf ? (const void*)ws->xb : (const void*)ws->x, md->w1[l], m, 4 * h, h, gl, s, ws->x3buf);
        }
        {
            ProfScope ps(s, MPIC_PHASE_W2);
            run_gemm(md, ws->ffn, md->w2[l], m, h, 4 * h, res, s, ws->x3buf);
        }
    }
    {
        ProfScope ps(s, MPIC_PHASE_LM_HEAD);
        if (logit_rows)  // batched requests: each request's last row, logits [request][V]
            for (size_t i = 0; i < logit_rows->size(); ++i)
                launch_lm_head(ws->x + (size_t)(*logit_rows)[i] * h, md->lm_head, md->dtype, c.vocab_size, h,
                               d_logits + i * c.vocab_size, s);
        else
            launch_lm_head(ws->x + (size_t)(m - 1) * h, md->lm_head, md->dtype, c.vocab_size, h, d_logits, s);
    }
    (void)e;
}

void check_ids(mpic_model_t md, const int32_t* ids, uint32_t m) {
    for (uint32_t i = 0; i < m; ++i)
        if (ids[i] < 0 || static_cast<uint32_t>(ids[i]) >= md->cfg.vocab_size)
            throw Error(MPIC_ERR_VALIDATION, "token id " + std::to_string(ids[i]) + " out of vocabulary");
}

// Host-pointer form: stage into pinned memory, run, bring logits back; synchronous.
void forward_host(mpic_model_t md, mpic_workspace_t ws, const int32_t* ids, const uint32_t* rows,
                  const uint32_t* pos, uint32_t m, mpic_kv_t kv, float* logits, cudaStream_t s,
                  float* hidden_out = nullptr, float* capture_out = nullptr) {
    MPIC_REQUIRE(ws && ws->model == md, MPIC_ERR_VALIDATION, "workspace belongs to another model");
    MPIC_REQUIRE(m > 0, MPIC_ERR_VALIDATION, "no tokens to prefill");
    MPIC_REQUIRE(m <= ws->max_rows, MPIC_ERR_VALIDATION, "more rows than the workspace holds");
    check_ids(md, ids, m);
    uint32_t max_pos = 0;
    for (uint32_t i = 0; i < m; ++i) {
        MPIC_REQUIRE(rows[i] < kv->T, MPIC_ERR_VALIDATION, "row index outside the cache");
        MPIC_REQUIRE(i == 0 || rows[i] > rows[i - 1], MPIC_ERR_CONTRACT, "rows must be ascending and unique");
        max_pos = std::max(max_pos, std::max(rows[i], pos[i]));
    }
    std::memcpy(ws->h_ids, ids, m * sizeof(int32_t));
    std::memcpy(ws->h_rows, rows, m * sizeof(uint32_t));
    std::memcpy(ws->h_pos, pos, m * sizeof(uint32_t));
    MPIC_CUDA(cudaMemcpyAsync(ws->d_ids, ws->h_ids, m * 4, cudaMemcpyHostToDevice, s));
    MPIC_CUDA(cudaMemcpyAsync(ws->d_rows, ws->h_rows, m * 4, cudaMemcpyHostToDevice, s));
    MPIC_CUDA(cudaMemcpyAsync(ws->d_pos, ws->h_pos, m * 4, cudaMemcpyHostToDevice, s));
    float* d_cap = nullptr;
    const size_t cap_elems = (size_t)md->cfg.n_layers * md->cfg.n_heads * kv->T * kv->T;
    if (capture_out) {
        MPIC_REQUIRE(md->dtype == MPIC_F32, MPIC_ERR_VALIDATION, "attention capture needs an fp32 model");
        MPIC_CUDA(cudaMallocAsync((void**)&d_cap, cap_elems * 4, s));
        MPIC_CUDA(cudaMemsetAsync(d_cap, 0, cap_elems * 4, s));
    }
    forward_rows(md, ws, ws->d_ids, ws->d_rows, ws->d_pos, m, max_pos, kv, ws->d_logits, s, {},
                 rows, d_cap);
    MPIC_CUDA(cudaMemcpyAsync(ws->h_logits, ws->d_logits, md->cfg.vocab_size * 4,
                              cudaMemcpyDeviceToHost, s));
    if (hidden_out)
        MPIC_CUDA(cudaMemcpyAsync(hidden_out, ws->x, (size_t)m * md->cfg.hidden_dim * 4,
                                  cudaMemcpyDeviceToHost, s));
    if (capture_out) {
        MPIC_CUDA(cudaMemcpyAsync(capture_out, d_cap, cap_elems * 4, cudaMemcpyDeviceToHost, s));
        MPIC_CUDA(cudaFreeAsync(d_cap, s));
    }
    MPIC_CUDA(cudaStreamSynchronize(s));
    std::memcpy(logits, ws->h_logits, md->cfg.vocab_size * sizeof(float));
}

// Host-side chunk placement: AsmChunk descriptors + per-chunk rerotation tables.
struct AsmPlan {
    std::vector<AsmChunk> chunks;
    std::vector<float2> tables;
    uint32_t n_tables = 0;
};

// src_ld / src_col0: source row width and first column (head-parallel slices); 0 / 0 =
// the destination's own width (T_dst_h = H_dst * D).
AsmPlan plan_assembly(const void* const* src_k, const void* const* src_v, const uint32_t* src_T,
                      const mpic_chunk_ref* chunks, uint32_t n, uint32_t T_dst, uint32_t D,
                      mpic_reposition rep, float rope_base, uint32_t T_dst_h = 0, uint32_t src_ld = 0,
                      uint32_t src_col0 = 0) {
    MPIC_REQUIRE(D % 2 == 0, MPIC_ERR_CONFIG, "head_dim must be even on the B200 path");
    AsmPlan p;
    p.chunks.resize(n);
    for (uint32_t i = 0; i < n; ++i) {
        const mpic_chunk_ref& c = chunks[i];
        MPIC_REQUIRE(c.dst_row0 + c.rows <= T_dst, MPIC_ERR_LINK, "chunk does not fit the request cache");
        MPIC_REQUIRE(c.src_row0 + c.rows <= src_T[i], MPIC_ERR_LINK, "chunk rows exceed the source entry");
        for (uint32_t j = 0; j < i; ++j)
            MPIC_REQUIRE(c.dst_row0 >= chunks[j].dst_row0 + chunks[j].rows ||
                             chunks[j].dst_row0 >= c.dst_row0 + c.rows,
                         MPIC_ERR_LINK, "chunks overlap in the request cache");
        AsmChunk a{};
        a.src_k = src_k ? src_k[i] : nullptr;
        a.src_v = src_v ? src_v[i] : nullptr;
        a.src_tokens = src_T[i];
        MPIC_REQUIRE(src_ld || T_dst_h, MPIC_ERR_VALIDATION, "assembly needs the destination row width");
        a.src_ld = src_ld ? src_ld : T_dst_h;
        a.src_col0 = src_col0;
        a.src_row0 = c.src_row0;
        a.dst_row0 = c.dst_row0;
        a.rows = c.rows;
        // rerotate_key from = position_base + j, to = start + j (linker.cpp:302-303):
        // the delta is constant over the chunk; from == to is a no-op (model.cpp:66-68).
        const double delta = static_cast<double>(c.dst_row0) -
                             (static_cast<double>(c.position_base) + static_cast<double>(c.src_row0));
        if (rep == MPIC_REROTATE && delta != 0.0) {
            a.rotate = 1;
            a.table = p.n_tables++;
            for (uint32_t q = 0; q + 1 < D; q += 2) {  // model.cpp:72-76
                const double freq = std::pow(static_cast<double>(rope_base), -static_cast<double>(q) / D);
                const double theta = delta * freq;
                p.tables.push_back(make_float2(static_cast<float>(std::cos(theta)),
                                               static_cast<float>(std::sin(theta))));
            }
        }
        p.chunks[i] = a;
    }
    // the assembly kernel binary-searches the chunk of each destination row
    std::sort(p.chunks.begin(), p.chunks.end(),
              [](const AsmChunk& a, const AsmChunk& b) { return a.dst_row0 < b.dst_row0; });
    return p;
}

// Copies a plan to a stream-ordered device buffer; returns (chunks, tables) pointers.
void* upload_plan(const AsmPlan& p, cudaStream_t s, const AsmChunk** dc, const float2** dt) {
    const size_t bytes_c = std::max<size_t>(1, p.chunks.size()) * sizeof(AsmChunk);
    const size_t bytes_t = std::max<size_t>(1, p.tables.size()) * sizeof(float2);
    void* dbuf = nullptr;
    MPIC_CUDA(cudaMallocAsync(&dbuf, bytes_c + bytes_t, s));
    if (!p.chunks.empty())
        MPIC_CUDA(cudaMemcpyAsync(dbuf, p.chunks.data(), p.chunks.size() * sizeof(AsmChunk),
                                  cudaMemcpyHostToDevice, s));
    if (!p.tables.empty())
        MPIC_CUDA(cudaMemcpyAsync((char*)dbuf + bytes_c, p.tables.data(), p.tables.size() * sizeof(float2),
                                  cudaMemcpyHostToDevice, s));
    *dc = static_cast<const AsmChunk*>(dbuf);
    *dt = reinterpret_cast<const float2*>((char*)dbuf + bytes_c);
    return dbuf;
}

void do_assemble(cudaStream_t s, const void* const* src_k, const void* const* src_v,
                 const uint32_t* src_T, mpic_dtype src_t, const mpic_chunk_ref* chunks,
                 uint32_t n, mpic_kv_t dst, mpic_reposition rep, int zero_gaps, float rope_base) {
    MPIC_REQUIRE(dst, MPIC_ERR_VALIDATION, "null destination cache");
    const AsmPlan p = plan_assembly(src_k, src_v, src_T, chunks, n, dst->T, dst->D, rep, rope_base, dst->H * dst->D);
    const AsmChunk* dc;
    const float2* dt;
    void* buf = upload_plan(p, s, &dc, &dt);
    {
        ProfScope ps(s, MPIC_PHASE_ASSEMBLE);
        launch_assemble(dc, n, dt, p.n_tables, src_t, dst->k, dst->v, dst->dtype, dst->L, dst->T,
                        dst->H, dst->D, zero_gaps, s);
    }
    MPIC_CUDA(cudaFreeAsync(buf, s));
}

// ---- request-level host logic -------------------------------------------------------
uint64_t fnv1a(const uint8_t* p, size_t n) {  // hash.h:18-25
    uint64_t h = 0xcbf29ce484222325ull;
    for (size_t i = 0; i < n; ++i) {
        h ^= p[i];
        h *= 0x100000001b3ull;
    }
    return h;
}
uint64_t mix64h(uint64_t x) {  // rng.h:10-17
    x ^= x >> 30;
    x *= 0xbf58476d1ce4e5b9ull;
    x ^= x >> 27;
    x *= 0x94d049bb133111ebull;
    x ^= x >> 31;
    return x;
}
uint64_t counter_hash_h(uint64_t seed, uint64_t stream, uint64_t i) {  // rng.h:19-24
    const uint64_t phi = 0x9e3779b97f4a7c15ull;
    uint64_t h = mix64h(seed + phi);
    h = mix64h(h ^ (stream + phi));
    return mix64h(h ^ (i + phi));
}

uint64_t fingerprint_of(const mpic_model_config* c);

void image_ids(const mpic_model_config* c, const uint8_t* hash32, uint32_t count, int32_t* out) {
    // model.cpp:148-156; the first two mixing rounds depend only on the key.
    const uint64_t key = fnv1a(hash32, 32) ^ fingerprint_of(c);
    const uint64_t phi = 0x9e3779b97f4a7c15ull;
    const uint64_t h1 = mix64h(mix64h(key + phi) ^ (0x696d67ull + phi));
    for (uint32_t i = 0; i < count; ++i)
        out[i] = static_cast<int32_t>(mix64h(h1 ^ (i + phi)) % c->vocab_size);
}

uint32_t prompt_tokens(const mpic_prompt* p) {
    MPIC_REQUIRE(p && p->n_segments > 0, MPIC_ERR_VALIDATION, "prompt needs at least one segment");
    uint32_t n = 0;
    for (uint32_t s = 0; s < p->n_segments; ++s) {
        MPIC_REQUIRE(p->lens[s] > 0, MPIC_ERR_VALIDATION,
                     p->kinds[s] == 0 ? "empty text segment" : "image segment token_count must be positive");
        n += p->lens[s];
    }
    return n;
}

uint32_t select_rows(const mpic_prompt* p, const mpic_policy* pol, uint32_t* out) {
    // linker.cpp:209-258; segments emit ascending indices, so the final sort is a no-op.
    const uint32_t n = prompt_tokens(p);
    if (pol->policy == MPIC_POLICY_ALL) {
        for (uint32_t i = 0; i < n; ++i) out[i] = i;
        return n;
    }
    if (pol->policy == MPIC_POLICY_PREFIX_ONLY) return 0;
    MPIC_REQUIRE(pol->policy == MPIC_POLICY_MPIC_K || pol->policy == MPIC_POLICY_TEXT_ONLY,
                 MPIC_ERR_VALIDATION, "unknown selection policy");
    const bool mk = pol->policy == MPIC_POLICY_MPIC_K;
    uint32_t budget = (mk && pol->global_budget) ? pol->k : 0, m = 0, at = 0;
    for (uint32_t s = 0; s < p->n_segments; ++s) {
        const uint32_t len = p->lens[s];
        if (p->kinds[s] == 0) {
            for (uint32_t i = 0; i < len; ++i) out[m++] = at + i;
        } else if (mk) {
            uint32_t take;
            if (pol->global_budget) {
                take = std::min(budget, len);
                budget -= take;
            } else {
                take = std::min(pol->k, len);
            }
            for (uint32_t i = 0; i < take; ++i) out[m++] = at + i;
        }
        at += len;
    }
    return m;
}

void flatten(const mpic_model_config* c, const mpic_prompt* p, int32_t* out) {
    // linker.cpp:160-172
    uint32_t ti = 0, hi = 0, at = 0;
    for (uint32_t s = 0; s < p->n_segments; ++s) {
        const uint32_t len = p->lens[s];
        if (p->kinds[s] == 0) {
            std::memcpy(out + at, p->text_ids + ti, len * sizeof(int32_t));
            ti += len;
        } else {
            image_ids(c, p->hashes + 32 * hi, len, out + at);
            ++hi;
        }
        at += len;
    }
}

// selective_prefill's contract checks (linker.cpp:319-340) for a freshly assembled cache
// whose Dummy slots are exactly the text segments.
void check_contract(const mpic_prompt* p, const uint32_t* sel, uint32_t m, uint32_t n) {
    MPIC_REQUIRE(m > 0, MPIC_ERR_CONTRACT, "selection mask is empty");
    MPIC_REQUIRE(sel[m - 1] < n, MPIC_ERR_CONTRACT, "selection mask index out of range");
    MPIC_REQUIRE(sel[m - 1] == n - 1, MPIC_ERR_CONTRACT, "final prompt token must be selected");
    uint32_t at = 0, j = 0;
    for (uint32_t s = 0; s < p->n_segments; ++s) {
        if (p->kinds[s] == 0)
            for (uint32_t i = at; i < at + p->lens[s]; ++i) {
                while (j < m && sel[j] < i) ++j;
                MPIC_REQUIRE(j < m && sel[j] == i, MPIC_ERR_CONTRACT,
                             "dummy slot " + std::to_string(i) + " not selected");
            }
        at += p->lens[s];
    }
}

struct RequestPlan {
    uint32_t n = 0, m = 0;
    std::vector<uint32_t> sel;
    std::vector<int32_t> ids_sel;
    std::vector<mpic_chunk_ref> refs;  // one per image segment, dst_row0 = segment start
};

RequestPlan plan_request(mpic_model_t md, const mpic_prompt* p, const mpic_policy* pol,
                         const uint32_t* position_bases) {
    RequestPlan r;
    r.n = prompt_tokens(p);
    r.sel.resize(r.n);
    r.m = select_rows(p, pol, r.sel.data());
    r.sel.resize(r.m);
    check_contract(p, r.sel.data(), r.m, r.n);
    std::vector<int32_t> flat(r.n);
    flatten(&md->cfg, p, flat.data());
    r.ids_sel.resize(r.m);
    for (uint32_t i = 0; i < r.m; ++i) r.ids_sel[i] = flat[r.sel[i]];
    uint32_t at = 0, img = 0;
    for (uint32_t s = 0; s < p->n_segments; ++s) {
        if (p->kinds[s] == 1) {
            mpic_chunk_ref c{};
            c.src_row0 = 0;
            c.dst_row0 = at;
            c.rows = p->lens[s];
            c.position_base = position_bases ? position_bases[img] : 0;
            r.refs.push_back(c);
            ++img;
        }
        at += p->lens[s];
    }
    return r;
}

void run_request(mpic_model_t md, mpic_workspace_t ws, const RequestPlan& r, mpic_kv_t linked,
                 float* logits, uint32_t* selected, uint32_t* m_out, cudaStream_t s,
                 const std::function<void(uint32_t)>& before_layer) {
    MPIC_REQUIRE(r.m <= ws->max_rows, MPIC_ERR_VALIDATION, "more rows than the workspace holds");
    check_ids(md, r.ids_sel.data(), r.m);
    std::memcpy(ws->h_ids, r.ids_sel.data(), r.m * sizeof(int32_t));
    std::memcpy(ws->h_rows, r.sel.data(), r.m * sizeof(uint32_t));
    MPIC_CUDA(cudaMemcpyAsync(ws->d_ids, ws->h_ids, r.m * 4, cudaMemcpyHostToDevice, s));
    MPIC_CUDA(cudaMemcpyAsync(ws->d_rows, ws->h_rows, r.m * 4, cudaMemcpyHostToDevice, s));
    forward_rows(md, ws, ws->d_ids, ws->d_rows, ws->d_rows, r.m, r.n - 1, linked, ws->d_logits, s,
                 before_layer, r.sel.data());
    MPIC_CUDA(cudaMemcpyAsync(ws->h_logits, ws->d_logits, md->cfg.vocab_size * 4,
                              cudaMemcpyDeviceToHost, s));
    MPIC_CUDA(cudaStreamSynchronize(s));
    std::memcpy(logits, ws->h_logits, md->cfg.vocab_size * sizeof(float));
    if (selected) std::memcpy(selected, r.sel.data(), r.m * sizeof(uint32_t));
    if (m_out) *m_out = r.m;
}

void check_linked(mpic_model_t md, mpic_kv_t linked, uint32_t n) {
    MPIC_REQUIRE(linked, MPIC_ERR_VALIDATION, "null linked cache");
    MPIC_REQUIRE(linked->T == n, MPIC_ERR_CONTRACT, "linked cache length does not match prompt");
    MPIC_REQUIRE(linked->L == md->cfg.n_layers && linked->H == md->cfg.n_heads &&
                     linked->D == md->cfg.head_dim && linked->dtype == md->dtype,
                 MPIC_ERR_VALIDATION, "linked cache shape does not match model");
}

// The compute lane of the loader paths (prepare, proj/src/transfer.cpp:119-140): an image
// chunk that is not in the tier (miss) or fails to load (fallback) is computed on the device
// as the reference's compute_entry does (transfer.cpp:41-58: prefill_extend of the image's
// token ids at position base 0), on its own stream and workspace, CONCURRENTLY with the
// request: the chunk prefill records an event after each layer, and layer l of the chunk is
// copied into the request's staging slot (cast to the slot dtype) once that event fires — so
// the request's layer l waits only for the chunk's layer l, not for the whole prefill.
struct MissLane {
    struct Job {
        uint32_t chunk = 0;
        mpic_kv_s kv;
        std::vector<cudaEvent_t> ev;  // ev[l]: layer l of the chunk is in kv
        std::vector<int32_t> ids;
        std::vector<uint32_t> rows;
        int32_t* d_ids = nullptr;
        uint32_t* d_rows = nullptr;
        size_t cap_bytes = 0;  // capacities of the (pooled) buffers
        uint32_t cap_rows = 0;
    };
    mpic_model_t md;
    mpic_workspace_t ws;
    std::vector<std::unique_ptr<Job>> jobs;

    MissLane(mpic_model_t m, mpic_workspace_t w) : md(m), ws(w) {}
    ~MissLane() {
        if (jobs.empty()) return;
        cudaStreamSynchronize(ws->miss_stream);
        cudaStreamSynchronize(ws->copy_stream);  // its layer copies read the chunk buffers
        for (auto& j : jobs) {  // back to the workspace's pool
            mpic_workspace_s::MissBuf b;
            b.k = j->kv.k;
            b.v = j->kv.v;
            b.d_ids = j->d_ids;
            b.d_rows = j->d_rows;
            b.bytes = j->cap_bytes;
            b.rows = j->cap_rows;
            b.ev = std::move(j->ev);
            ws->miss_pool.push_back(std::move(b));
        }
    }
    Job* find(uint32_t chunk) const {
        for (auto& j : jobs)
            if (j->chunk == chunk) return j.get();
        return nullptr;
    }
    // Start computing chunk `chunk` (image hash, T tokens). `after`: stream whose work so far
    // must precede the lane (the request's plan uploads; nothing of the chunk depends on it,
    // but the aux workspace must not race an earlier user).
    Job* start(uint32_t chunk, const uint8_t* hash32, uint32_t T) {
        if (Job* j = find(chunk)) return j;
        const mpic_model_config& c = md->cfg;
        if (!ws->miss_stream) MPIC_CUDA(cudaStreamCreateWithFlags(&ws->miss_stream, cudaStreamNonBlocking));
        if (!ws->aux || ws->aux->max_rows < T) {
            if (ws->aux) {
                MPIC_CUDA(cudaStreamSynchronize(ws->miss_stream));
                mpic_workspace_destroy(ws->aux);
                ws->aux = nullptr;
            }
            const uint32_t launches = g_launches;  // the nested API call resets the counter
            const int rc = mpic_workspace_create(md, T, T, &ws->aux);
            g_launches = launches;
            if (rc != MPIC_OK) throw Error(rc, std::string("compute lane workspace: ") + g_last_error);
        }
        auto job = std::make_unique<Job>();
        Job& j = *job;
        j.chunk = chunk;
        j.kv.L = c.n_layers;
        j.kv.T = T;
        j.kv.H = c.n_heads;
        j.kv.D = c.head_dim;
        j.kv.dtype = md->dtype;
        j.kv.device = md->device;
        const size_t bytes = j.kv.elems() * esz(md->dtype);
        auto& pool = ws->miss_pool;
        size_t pick = pool.size();
        for (size_t i = 0; i < pool.size(); ++i)  // the smallest pooled buffer set that fits
            if (pool[i].bytes >= bytes && pool[i].rows >= T && pool[i].ev.size() >= c.n_layers &&
                (pick == pool.size() || pool[i].bytes < pool[pick].bytes))
                pick = i;
        if (pick < pool.size()) {
            mpic_workspace_s::MissBuf& b = pool[pick];
            j.kv.k = b.k;
            j.kv.v = b.v;
            j.d_ids = b.d_ids;
            j.d_rows = b.d_rows;
            j.cap_bytes = b.bytes;
            j.cap_rows = b.rows;
            j.ev = std::move(b.ev);
            pool.erase(pool.begin() + (ptrdiff_t)pick);
        } else {
            MPIC_CUDA(cudaMalloc(&j.kv.k, bytes));
            MPIC_CUDA(cudaMalloc(&j.kv.v, bytes));
            MPIC_CUDA(cudaMalloc(&j.d_ids, T * sizeof(int32_t)));
            MPIC_CUDA(cudaMalloc(&j.d_rows, T * sizeof(uint32_t)));
            j.cap_bytes = bytes;
            j.cap_rows = T;
        }
        j.ids.resize(T);
        image_ids(&c, hash32, T, j.ids.data());  // model.cpp:148-156
        j.rows.resize(T);
        for (uint32_t i = 0; i < T; ++i) j.rows[i] = i;  // rows == positions: base 0
        while (j.ev.size() < c.n_layers) {
            cudaEvent_t e;
            MPIC_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            j.ev.push_back(e);
        }
        cudaStream_t st = ws->miss_stream;
        MPIC_CUDA(cudaMemcpyAsync(j.d_ids, j.ids.data(), T * 4, cudaMemcpyHostToDevice, st));
        MPIC_CUDA(cudaMemcpyAsync(j.d_rows, j.rows.data(), T * 4, cudaMemcpyHostToDevice, st));
        jobs.push_back(std::move(job));
        forward_rows(md, ws->aux, j.d_ids, j.d_rows, j.d_rows, T, T - 1, &j.kv, ws->aux->d_logits, st,
                     [&](uint32_t l) {
                         if (l) MPIC_CUDA(cudaEventRecord(j.ev[l - 1], st));
                     },
                     j.rows.data());
        MPIC_CUDA(cudaEventRecord(j.ev[c.n_layers - 1], st));
        return &j;
    }
    // Layer l of a computed chunk -> dst_k / dst_v (rows [0, T) x h, dtype dt) on stream cs.
    void copy_layer(const Job& j, uint32_t l, void* dst_k, void* dst_v, mpic_dtype dt, cudaStream_t cs) const {
        const size_t cnt = (size_t)j.kv.T * j.kv.H * j.kv.D, es = esz(j.kv.dtype);
        MPIC_CUDA(cudaStreamWaitEvent(cs, j.ev[l], 0));
        const char* sk = static_cast<const char*>(j.kv.k) + l * cnt * es;
        const char* sv = static_cast<const char*>(j.kv.v) + l * cnt * es;
        if (dt == j.kv.dtype) {
            MPIC_CUDA(cudaMemcpyAsync(dst_k, sk, cnt * es, cudaMemcpyDeviceToDevice, cs));
            MPIC_CUDA(cudaMemcpyAsync(dst_v, sv, cnt * es, cudaMemcpyDeviceToDevice, cs));
        } else if (dt == MPIC_F32) {
            launch_bf16_to_f32(reinterpret_cast<const __nv_bfloat16*>(sk), static_cast<float*>(dst_k), cnt, cs);
            launch_bf16_to_f32(reinterpret_cast<const __nv_bfloat16*>(sv), static_cast<float*>(dst_v), cnt, cs);
        } else {
            launch_f32_to_bf16(reinterpret_cast<const float*>(sk), static_cast<__nv_bfloat16*>(dst_k), cnt, cs);
            launch_f32_to_bf16(reinterpret_cast<const float*>(sv), static_cast<__nv_bfloat16*>(dst_v), cnt, cs);
        }
    }
};

// Image hashes of a prompt, one per image segment (in segment order).
std::vector<const uint8_t*> image_hashes(const mpic_prompt* p) {
    std::vector<const uint8_t*> out;
    for (uint32_t s = 0, hi = 0; s < p->n_segments; ++s)
        if (p->kinds[s] == 1) out.push_back(p->hashes + 32 * hi++);
    return out;
}

}  // namespace

extern "C" uint64_t mpic_config_fingerprint(const mpic_model_config* c);
namespace {
uint64_t fingerprint_of(const mpic_model_config* c) { return mpic_config_fingerprint(c); }
}  // namespace

extern "C" {

const char* mpic_last_error(void) { return g_last_error.c_str(); }
const char* mpic_version(void) { return "mpic-b200 0.1 (sm_100a)"; }
uint32_t mpic_last_launch_count(void) { return g_launches; }

int mpic_config_validate(const mpic_model_config* cfg) {
    API_BEGIN
    validate_cfg(cfg);
    API_END
}

uint64_t mpic_config_fingerprint(const mpic_model_config* c) {
    // ModelConfig::fingerprint (proj/src/config.cpp:30-47)
    uint32_t rb;
    std::memcpy(&rb, &c->rope_base, 4);
    const uint64_t f[8] = {c->n_layers, c->n_heads, c->head_dim, c->hidden_dim,
                           c->vocab_size, c->image_token_count, rb, c->seed};
    uint64_t h = 0xcbf29ce484222325ull;
    for (uint64_t v : f)
        for (int b = 0; b < 8; ++b) {
            h ^= static_cast<uint8_t>(v >> (8 * b));
            h *= 0x100000001b3ull;
        }
    return h;
}

int mpic_model_create(const mpic_model_config* cfg, int device, mpic_dtype dtype, mpic_model_t* out) {
    mpic_model_t m = nullptr;
    API_BEGIN
    validate_cfg(cfg);
    validate_device_cfg(cfg);
    set_device(device);
    m = new mpic_model_s();
    m->cfg = *cfg;
    m->device = device;
    m->dtype = dtype;
    alloc_model(m);
    const size_t h = cfg->hidden_dim, V = cfg->vocab_size;
    const float scale = 1.0f / std::sqrt(static_cast<float>(h));  // model.cpp:106
    const size_t e = esz(dtype);
    cudaStream_t s = 0;
    launch_synth(cfg->seed, 100, 0, V * h, 1.0f, m->emb, MPIC_F32, s);
    launch_synth(cfg->seed, 101, 0, V * h, scale, m->lm_head, dtype, s);
    for (uint32_t l = 0; l < cfg->n_layers; ++l) {
        launch_synth(cfg->seed, 1, l, h * h, scale, m->wqkv[l], dtype, s);
        launch_synth(cfg->seed, 2, l, h * h, scale, (char*)m->wqkv[l] + h * h * e, dtype, s);
        launch_synth(cfg->seed, 3, l, h * h, scale, (char*)m->wqkv[l] + 2 * h * h * e, dtype, s);
        launch_synth(cfg->seed, 4, l, h * h, scale, m->wo[l], dtype, s);
        launch_synth(cfg->seed, 5, l, 4 * h * h, scale, m->w1[l], dtype, s);
        launch_synth(cfg->seed, 6, l, 4 * h * h, scale, m->w2[l], dtype, s);
    }
    ensure_rope(m, 1, s);
    prepare_x3(m, s);
    MPIC_CUDA(cudaDeviceSynchronize());
    *out = m;
    m = nullptr;
    API_END
}

int mpic_model_upload(const mpic_model_config* cfg, int device, mpic_dtype dtype,
                      const float* embedding, const float* lm_head, const float* const* layer_w,
                      mpic_model_t* out) {
    mpic_model_t m = nullptr;
    API_BEGIN
    validate_cfg(cfg);
    validate_device_cfg(cfg);
    set_device(device);
    m = new mpic_model_s();
    m->cfg = *cfg;
    m->device = device;
    m->dtype = dtype;
    alloc_model(m);
    cudaStream_t s = 0;
    for (int which = 0; which < 8; ++which) {
        const uint32_t nl = which < 2 ? 1 : cfg->n_layers;
        for (uint32_t l = 0; l < nl; ++l) {
            size_t cnt;
            void* dst = weight_ptr(m, which, l, &cnt);
            const float* src = which == 0 ? embedding : which == 1 ? lm_head : layer_w[6 * l + (which - 2)];
            upload_cast(dst, which == 0 ? MPIC_F32 : dtype, src, cnt, s);
        }
    }
    ensure_rope(m, 1, s);
    prepare_x3(m, s);
    MPIC_CUDA(cudaDeviceSynchronize());
    *out = m;
    m = nullptr;
    API_END
}

int mpic_model_destroy(mpic_model_t model) {
    API_BEGIN
    free_model(model);
    API_END
}

int mpic_model_config_get(mpic_model_t model, mpic_model_config* out) {
    API_BEGIN
    *out = model->cfg;
    API_END
}

mpic_dtype mpic_model_dtype(mpic_model_t model) { return model->dtype; }
int mpic_model_device(mpic_model_t model) { return model->device; }

int mpic_model_download_weight(mpic_model_t m, int which, uint32_t layer, float* out) {
    API_BEGIN
    MPIC_CUDA(cudaSetDevice(m->device));
    size_t cnt;
    void* src = weight_ptr(m, which, layer, &cnt);
    download_cast(out, src, which == 0 ? MPIC_F32 : m->dtype, cnt, 0);
    API_END
}

int mpic_kv_alloc(uint32_t L, uint32_t T, uint32_t H, uint32_t D, mpic_dtype dtype, int device,
                  mpic_kv_t* out) {
    mpic_kv_t kv = nullptr;
    API_BEGIN
    MPIC_REQUIRE(L && H && D, MPIC_ERR_VALIDATION, "degenerate cache shape");
    set_device(device);
    kv = new mpic_kv_s();
    kv->L = L; kv->T = T; kv->H = H; kv->D = D;
    kv->dtype = dtype;
    kv->device = device;
    const size_t bytes = std::max<size_t>(1, kv->elems()) * esz(dtype);
    MPIC_CUDA(cudaMalloc(&kv->k, bytes));
    MPIC_CUDA(cudaMalloc(&kv->v, bytes));
    *out = kv;
    kv = nullptr;
    API_END
}

int mpic_kv_free(mpic_kv_t kv) {
    API_BEGIN
    if (kv) {
        cudaSetDevice(kv->device);
        cudaFree(kv->k);
        cudaFree(kv->v);
        delete kv;
    }
    API_END
}

int mpic_kv_shape(mpic_kv_t kv, uint32_t* shape4, mpic_dtype* dtype) {
    API_BEGIN
    shape4[0] = kv->L; shape4[1] = kv->T; shape4[2] = kv->H; shape4[3] = kv->D;
    if (dtype) *dtype = kv->dtype;
    API_END
}

int mpic_kv_device_ptrs(mpic_kv_t kv, void** k, void** v) {
    API_BEGIN
    *k = kv->k;
    *v = kv->v;
    API_END
}

int mpic_kv_upload(mpic_kv_t kv, const float* k, const float* v, void* stream) {
    API_BEGIN
    MPIC_CUDA(cudaSetDevice(kv->device));
    upload_cast(kv->k, kv->dtype, k, kv->elems(), (cudaStream_t)stream);
    upload_cast(kv->v, kv->dtype, v, kv->elems(), (cudaStream_t)stream);
    API_END
}

int mpic_kv_download_rows(mpic_kv_t kv, const uint32_t* rows, uint32_t n_rows, float* k, float* v,
                          void* stream) {
    API_BEGIN
    MPIC_CUDA(cudaSetDevice(kv->device));
    cudaStream_t s = (cudaStream_t)stream;
    if (n_rows == 0) return MPIC_OK;
    const size_t h = (size_t)kv->H * kv->D, per = (size_t)kv->L * n_rows * h;
    for (uint32_t i = 0; i < n_rows; ++i)
        MPIC_REQUIRE(rows[i] < kv->T, MPIC_ERR_VALIDATION, "row index outside the cache");
    uint32_t* d_rows = nullptr;
    float* stage = nullptr;
    MPIC_CUDA(cudaMallocAsync((void**)&d_rows, n_rows * sizeof(uint32_t), s));
    MPIC_CUDA(cudaMallocAsync((void**)&stage, 2 * per * sizeof(float), s));
    MPIC_CUDA(cudaMemcpyAsync(d_rows, rows, n_rows * sizeof(uint32_t), cudaMemcpyHostToDevice, s));
    launch_gather_rows(kv->k, kv->v, kv->dtype, kv->L, kv->T, (uint32_t)h, d_rows, n_rows, stage, stage + per, s);
    std::vector<float> host(2 * per);
    MPIC_CUDA(cudaMemcpyAsync(host.data(), stage, 2 * per * sizeof(float), cudaMemcpyDeviceToHost, s));
    MPIC_CUDA(cudaFreeAsync(d_rows, s));
    MPIC_CUDA(cudaFreeAsync(stage, s));
    MPIC_CUDA(cudaStreamSynchronize(s));
    for (uint32_t l = 0; l < kv->L; ++l)
        for (uint32_t i = 0; i < n_rows; ++i) {
            const size_t src = ((size_t)l * n_rows + i) * h, dst = ((size_t)l * kv->T + rows[i]) * h;
            if (k) std::memcpy(k + dst, host.data() + src, h * sizeof(float));
            if (v) std::memcpy(v + dst, host.data() + per + src, h * sizeof(float));
        }
    API_END
}

int mpic_kv_download(mpic_kv_t kv, float* k, float* v, void* stream) {
    API_BEGIN
    MPIC_CUDA(cudaSetDevice(kv->device));
    if (k) download_cast(k, kv->k, kv->dtype, kv->elems(), (cudaStream_t)stream);
    if (v) download_cast(v, kv->v, kv->dtype, kv->elems(), (cudaStream_t)stream);
    API_END
}

int mpic_kv_zero_rows(mpic_kv_t kv, uint32_t row0, uint32_t rows, void* stream) {
    API_BEGIN
    MPIC_REQUIRE(row0 + rows <= kv->T, MPIC_ERR_VALIDATION, "rows outside the cache");
    MPIC_CUDA(cudaSetDevice(kv->device));
    const size_t row_b = (size_t)kv->H * kv->D * esz(kv->dtype);
    const size_t plane = (size_t)kv->T * row_b;
    if (rows) {
        MPIC_CUDA(cudaMemset2DAsync((char*)kv->k + row0 * row_b, plane, 0, rows * row_b, kv->L, (cudaStream_t)stream));
        MPIC_CUDA(cudaMemset2DAsync((char*)kv->v + row0 * row_b, plane, 0, rows * row_b, kv->L, (cudaStream_t)stream));
    }
    API_END
}

int mpic_assemble(void* stream, const mpic_chunk_ref* chunks, uint32_t n_chunks, mpic_kv_t dst,
                  mpic_reposition reposition, float rope_base, int zero_gaps) {
    API_BEGIN
    MPIC_REQUIRE(dst, MPIC_ERR_VALIDATION, "null destination cache");
    MPIC_CUDA(cudaSetDevice(dst->device));
    std::vector<const void*> ks(n_chunks), vs(n_chunks);
    std::vector<uint32_t> ts(n_chunks);
    mpic_dtype st = dst->dtype;
    for (uint32_t i = 0; i < n_chunks; ++i) {
        const mpic_kv_t s = chunks[i].src;
        MPIC_REQUIRE(s, MPIC_ERR_LINK, "null chunk");
        MPIC_REQUIRE(s->L == dst->L && s->H == dst->H && s->D == dst->D, MPIC_ERR_LINK,
                     "entry tensor shape does not match model");
        MPIC_REQUIRE(i == 0 || s->dtype == st, MPIC_ERR_VALIDATION, "mixed chunk dtypes");
        st = s->dtype;
        ks[i] = s->k;
        vs[i] = s->v;
        ts[i] = s->T;
    }
    do_assemble((cudaStream_t)stream, ks.data(), vs.data(), ts.data(), st, chunks, n_chunks, dst,
                reposition, zero_gaps, rope_base);
    API_END
}

int mpic_assemble_raw(void* stream, const void* const* src_k, const void* const* src_v,
                      const uint32_t* src_tokens, mpic_dtype src_dtype, const mpic_chunk_ref* chunks,
                      uint32_t n_chunks, mpic_kv_t dst, mpic_reposition reposition, float rope_base,
                      int zero_gaps) {
    API_BEGIN
    MPIC_REQUIRE(dst, MPIC_ERR_VALIDATION, "null destination cache");
    MPIC_CUDA(cudaSetDevice(dst->device));
    do_assemble((cudaStream_t)stream, src_k, src_v, src_tokens, src_dtype, chunks, n_chunks, dst,
                reposition, zero_gaps, rope_base);
    API_END
}

int mpic_workspace_create(mpic_model_t md, uint32_t max_rows, uint32_t max_ctx, mpic_workspace_t* out) {
    mpic_workspace_t ws = nullptr;
    API_BEGIN
    MPIC_REQUIRE(md && max_rows > 0, MPIC_ERR_VALIDATION, "bad workspace request");
    MPIC_CUDA(cudaSetDevice(md->device));
    {
        // Stream-ordered allocations of the request paths (plan uploads, batch logits) come
        // from the device's default pool: keep its memory instead of returning it to the
        // driver at every synchronisation (re-mapping it per request takes the driver lock
        // and stalled single requests by 100s of ms under load)
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, md->device) == cudaSuccess) {
            uint64_t keep = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        }
    }
    ws = new mpic_workspace_s();
    ws->model = md;
    ws->max_rows = max_rows;
    ws->max_ctx = max_ctx;
    ws->m_pad = (max_rows + 127) / 128 * 128;
    const size_t h = md->cfg.hidden_dim, mp = ws->m_pad;
    const size_t e = esz(md->dtype);
    ws->d_ids = dmalloc<int32_t>(mp);
    ws->d_rows = dmalloc<uint32_t>(mp);
    ws->d_pos = dmalloc<uint32_t>(mp);
    ws->d_start = dmalloc<uint32_t>(mp);
    ws->x = dmalloc<float>(mp * h);
    ws->rope_tok = dmalloc<float2>(mp * (md->cfg.head_dim / 2));
    ws->xb = dmalloc<__nv_bfloat16>(mp * h);
    MPIC_CUDA(cudaMalloc(&ws->q, mp * h * e));
    MPIC_CUDA(cudaMalloc(&ws->attn, mp * h * e));
    MPIC_CUDA(cudaMalloc(&ws->ffn, mp * 4 * h * e));
    // Padding rows of the GEMM A operands are read (never written back): keep them finite.
    MPIC_CUDA(cudaMemset(ws->xb, 0, mp * h * 2));
    MPIC_CUDA(cudaMemset(ws->attn, 0, mp * h * e));
    MPIC_CUDA(cudaMemset(ws->ffn, 0, mp * 4 * h * e));
    ws->d_logits = dmalloc<float>(md->cfg.vocab_size);
    if (md->dtype == MPIC_BF16) {
        ws->partial_cap = 8 * mp * h;
        ws->partial = dmalloc<float>(ws->partial_cap);
    }
    if (!md->x3w.empty()) ws->x3buf = dmalloc<float>(2 * mp * 4 * h);
    MPIC_CUDA(cudaMallocHost(&ws->h_ids, mp * 4));
    MPIC_CUDA(cudaMallocHost(&ws->h_rows, mp * 4));
    MPIC_CUDA(cudaMallocHost(&ws->h_pos, mp * 4));
    MPIC_CUDA(cudaMallocHost(&ws->h_start, mp * 4));
    MPIC_CUDA(cudaMallocHost(&ws->h_logits, md->cfg.vocab_size * 4));
    MPIC_CUDA(cudaStreamCreateWithFlags(&ws->copy_stream, cudaStreamNonBlocking));
    for (int i = 0; i < 2; ++i) {
        MPIC_CUDA(cudaEventCreateWithFlags(&ws->ev_ready[i], cudaEventDisableTiming));
        MPIC_CUDA(cudaEventCreateWithFlags(&ws->ev_free[i], cudaEventDisableTiming));
    }
    *out = ws;
    ws = nullptr;
    API_END
}

int mpic_workspace_destroy(mpic_workspace_t ws) {
    API_BEGIN
    if (ws) {
        cudaSetDevice(ws->model->device);
        cudaFree(ws->d_ids); cudaFree(ws->d_rows); cudaFree(ws->d_pos); cudaFree(ws->d_start);
        cudaFree(ws->x); cudaFree(ws->rope_tok); cudaFree(ws->xb); cudaFree(ws->q); cudaFree(ws->attn); cudaFree(ws->ffn);
        cudaFree(ws->d_logits);
        cudaFree(ws->partial);
        cudaFree(ws->x3buf);
        cudaFreeHost(ws->h_ids); cudaFreeHost(ws->h_rows); cudaFreeHost(ws->h_pos); cudaFreeHost(ws->h_start);
        cudaFreeHost(ws->h_logits);
        for (int i = 0; i < 2; ++i) {
            cudaFree(ws->stage[i]);
            if (ws->ev_ready[i]) cudaEventDestroy(ws->ev_ready[i]);
            if (ws->ev_free[i]) cudaEventDestroy(ws->ev_free[i]);
        }
        if (ws->copy_stream) cudaStreamDestroy(ws->copy_stream);
        cudaFree(ws->d_units);
        cudaFree(ws->d_comb);
        cudaFree(ws->d_comb_cnt);
        cudaFree(ws->part_o);
        cudaFree(ws->part_ml);
        cudaFreeHost(ws->h_plan);
        cudaFreeHost(ws->h_asm);
        cudaFree(ws->d_asm);
        if (ws->ev_plan) cudaEventDestroy(ws->ev_plan);
        if (ws->graph) cudaGraphExecDestroy(ws->graph);
        for (int i = 0; i < 3; ++i) {
            cudaFreeHost(ws->pin[i]);
            if (ws->ev_pin[i]) cudaEventDestroy(ws->ev_pin[i]);
        }
        for (cudaEvent_t e : ws->ev_asm) cudaEventDestroy(e);
        if (ws->ev_asm_in) cudaEventDestroy(ws->ev_asm_in);
        if (ws->asm_stream) cudaStreamDestroy(ws->asm_stream);
        if (ws->miss_stream) {
            cudaStreamSynchronize(ws->miss_stream);
            cudaStreamDestroy(ws->miss_stream);
        }
        if (ws->aux) mpic_workspace_destroy(ws->aux);
        for (auto& b : ws->miss_pool) {
            cudaFree(b.k);
            cudaFree(b.v);
            cudaFree(b.d_ids);
            cudaFree(b.d_rows);
            for (cudaEvent_t e : b.ev) cudaEventDestroy(e);
        }
        cudaFree(ws->hp_partial);
        cudaFree(ws->hp_reduced);
        if (ws->hp_graph) cudaGraphExecDestroy(ws->hp_graph);
        delete ws;
    }
    API_END
}

int mpic_selective_prefill(mpic_model_t model, mpic_workspace_t ws, const int32_t* ids,
                           const uint32_t* rows, uint32_t m, mpic_kv_t kv, float* logits, void* stream) {
    API_BEGIN
    MPIC_CUDA(cudaSetDevice(model->device));
    // selective_core rotates each row at its own global index (linker.cpp:67-70).
    forward_host(model, ws, ids, rows, rows, m, kv, logits, (cudaStream_t)stream);
    API_END
}

int mpic_prefill_extend(mpic_model_t model, mpic_workspace_t ws, const int32_t* ids, uint32_t m,
                        uint32_t start, uint32_t position_base, mpic_kv_t kv, float* logits, void* stream) {
    API_BEGIN
    MPIC_CUDA(cudaSetDevice(model->device));
    MPIC_REQUIRE(start + m <= kv->T, MPIC_ERR_VALIDATION, "cache too short for the new rows");
    std::vector<uint32_t> rows(m), pos(m);
    for (uint32_t i = 0; i < m; ++i) {  // model.cpp:253
        rows[i] = start + i;
        pos[i] = position_base + start + i;
    }
    forward_host(model, ws, ids, rows.data(), pos.data(), m, kv, logits, (cudaStream_t)stream);
    API_END
}

int mpic_forward_rows(mpic_model_t model, mpic_workspace_t ws, const int32_t* ids,
                      const uint32_t* rows, const uint32_t* rope_pos, uint32_t m, mpic_kv_t kv,
                      float* logits, float* hidden_out, float* attn_capture, void* stream) {
    API_BEGIN
    MPIC_CUDA(cudaSetDevice(model->device));
    forward_host(model, ws, ids, rows, rope_pos, m, kv, logits, (cudaStream_t)stream, hidden_out,
                 attn_capture);
    API_END
}

int mpic_layer0_keys(mpic_model_t model, mpic_workspace_t ws, const int32_t* ids,
                     const uint32_t* positions, uint32_t m, float* out, void* stream) {
    API_BEGIN
    MPIC_CUDA(cudaSetDevice(model->device));
    MPIC_REQUIRE(ws && ws->model == model && m <= ws->max_rows, MPIC_ERR_VALIDATION, "bad workspace");
    if (m == 0) return MPIC_OK;
    cudaStream_t s = (cudaStream_t)stream;
    check_ids(model, ids, m);
    const mpic_model_config& c = model->cfg;
    const uint32_t h = c.hidden_dim;
    uint32_t max_pos = 0;
    for (uint32_t i = 0; i < m; ++i) max_pos = std::max(max_pos, positions[i]);
    ensure_rope(model, max_pos + 1, s);
    std::vector<uint32_t> rows(m);
    for (uint32_t i = 0; i < m; ++i) rows[i] = i;
    std::memcpy(ws->h_ids, ids, m * 4);
    std::memcpy(ws->h_rows, rows.data(), m * 4);
    std::memcpy(ws->h_pos, positions, m * 4);
    MPIC_CUDA(cudaMemcpyAsync(ws->d_ids, ws->h_ids, m * 4, cudaMemcpyHostToDevice, s));
    MPIC_CUDA(cudaMemcpyAsync(ws->d_rows, ws->h_rows, m * 4, cudaMemcpyHostToDevice, s));
    MPIC_CUDA(cudaMemcpyAsync(ws->d_pos, ws->h_pos, m * 4, cudaMemcpyHostToDevice, s));
    const bool bf = model->dtype == MPIC_BF16;
    launch_embed(model->emb, ws->d_ids, m, h, ws->x, bf ? ws->xb : nullptr, s);
    const size_t e = esz(model->dtype);
    void* kbuf = nullptr;
    void* vbuf = nullptr;
    MPIC_CUDA(cudaMallocAsync(&kbuf, (size_t)m * h * e, s));
    MPIC_CUDA(cudaMallocAsync(&vbuf, (size_t)m * h * e, s));
    EpiParams qkv;  // layer-0 Q/K/V with K rotated at `positions` (linker.cpp:493-499)
    qkv.mode = EPI_QKV;
    qkv.q = ws->q;
    qkv.kv_k = kbuf;
    qkv.kv_v = vbuf;
    qkv.kv_rows = ws->d_rows;
    qkv.rope_pos = ws->d_pos;
    qkv.rope = model->rope;
    qkv.hidden = h;
    qkv.head_dim = c.head_dim;
    run_gemm(model, bf ? (const void*)ws->xb : (const void*)ws->x, model->wqkv[0], m, 3 * h, h, qkv, s);
    download_cast(out, kbuf, model->dtype, (size_t)m * h, s);
    MPIC_CUDA(cudaFreeAsync(kbuf, s));
    MPIC_CUDA(cudaFreeAsync(vbuf, s));
    MPIC_CUDA(cudaStreamSynchronize(s));
    API_END
}

int mpic_forward_rows_async(mpic_model_t model, mpic_workspace_t ws, const int32_t* d_ids,
                            const uint32_t* d_rows, const uint32_t* d_rope_pos, uint32_t m,
                            uint32_t max_pos, mpic_kv_t kv, float* d_logits, void* stream) {
    API_BEGIN
    MPIC_CUDA(cudaSetDevice(model->device));
    forward_rows(model, ws, d_ids, d_rows, d_rope_pos, m, max_pos, kv, d_logits, (cudaStream_t)stream);
    API_END
}


int mpic_image_token_ids(const mpic_model_config* cfg, const uint8_t* hash32, uint32_t count,
                         int32_t* out) {
    API_BEGIN
    validate_cfg(cfg);
    image_ids(cfg, hash32, count, out);
    API_END
}

int mpic_select_tokens(const mpic_prompt* prompt, const mpic_policy* policy, uint32_t* out,
                       uint32_t* m) {
    API_BEGIN
    *m = select_rows(prompt, policy, out);
    API_END
}

int mpic_flatten_ids(const mpic_model_config* cfg, const mpic_prompt* prompt, int32_t* out) {
    API_BEGIN
    prompt_tokens(prompt);
    flatten(cfg, prompt, out);
    API_END
}

int mpic_request_prefill(mpic_model_t model, mpic_workspace_t ws, const mpic_prompt* prompt,
                         const mpic_policy* policy, const mpic_kv_t* chunks,
                         mpic_reposition reposition, const uint32_t* position_bases,
                         mpic_kv_t linked, float* logits, uint32_t* selected, uint32_t* m_out,
                         void* stream) {
    API_BEGIN
    MPIC_CUDA(cudaSetDevice(model->device));
    cudaStream_t s = (cudaStream_t)stream;
    MPIC_REQUIRE(ws && ws->model == model, MPIC_ERR_VALIDATION, "workspace belongs to another model");
    // ---- host planning (select, contract, assembly and attention plans, staging) ----
    const RequestPlan r = plan_request(model, prompt, policy, position_bases);
    check_linked(model, linked, r.n);
    MPIC_REQUIRE(r.m <= ws->max_rows, MPIC_ERR_VALIDATION, "more rows than the workspace holds");
    check_ids(model, r.ids_sel.data(), r.m);
    const uint32_t n_img = (uint32_t)r.refs.size();
    std::vector<const void*> ks(n_img), vs(n_img);
    std::vector<uint32_t> ts(n_img);
    for (uint32_t i = 0; i < n_img; ++i) {
        const mpic_kv_t c = chunks[i];
        MPIC_REQUIRE(c, MPIC_ERR_LINK, "no fetched entry for image segment");
        MPIC_REQUIRE(c->T == r.refs[i].rows, MPIC_ERR_LINK, "token_count mismatch for image segment");
        MPIC_REQUIRE(c->L == linked->L && c->H == linked->H && c->D == linked->D, MPIC_ERR_LINK,
                     "entry tensor shape does not match model");
        MPIC_REQUIRE(c->dtype == chunks[0]->dtype, MPIC_ERR_VALIDATION, "mixed chunk dtypes");
        ks[i] = c->k;
        vs[i] = c->v;
        ts[i] = c->T;
    }
    const mpic_dtype src_t = n_img ? chunks[0]->dtype : model->dtype;
    const AsmPlan ap = plan_assembly(ks.data(), vs.data(), ts.data(), r.refs.data(), n_img, linked->T, linked->D,
                                     reposition, model->cfg.rope_base, linked->H * linked->D);
    ensure_rope(model, r.n, s);
    if (use_tc_attention(model)) prepare_attn_plan(ws, r.sel.data(), r.m, r.n - 1, model->cfg.n_heads);
    std::memcpy(ws->h_ids, r.ids_sel.data(), r.m * sizeof(int32_t));
    std::memcpy(ws->h_rows, r.sel.data(), r.m * sizeof(uint32_t));
    // linking inside attention: chunk blocks skip the assembly and are stored by attention
    std::vector<uint32_t> link_blk;
    std::vector<uint16_t> link_wtile;
    std::vector<uint8_t> link_skip;
    const bool link = attn_link_enabled() && use_tc_attention(model) && linked->dtype == MPIC_BF16 &&
                      src_t == MPIC_BF16 && n_img > 0 && n_img <= kMaxLinkChunks && ap.n_tables == 0 &&
                      plan_attn_link(r.refs, r.sel.data(), r.m, r.n, link_blk, link_wtile, link_skip);
    const size_t bytes_c = std::max<size_t>(1, ap.chunks.size()) * sizeof(AsmChunk);
    const size_t bytes_t = std::max<size_t>(1, ap.tables.size()) * sizeof(float2);
    const size_t off_l = (bytes_c + bytes_t + 63) & ~size_t(63);
    const size_t bytes_l = link ? sizeof(AttnLink) + link_blk.size() * 6 : 0;
    const size_t off_s = off_l + ((bytes_l + 63) & ~size_t(63));
    const size_t bytes_all = off_s + link_skip.size();
    if (ws->asm_cap < bytes_all) {
        ++ws->gen;
        MPIC_CUDA(cudaDeviceSynchronize());
        cudaFreeHost(ws->h_asm);
        cudaFree(ws->d_asm);
        ws->h_asm = ws->d_asm = nullptr;
        ws->asm_cap = 0;
        MPIC_CUDA(cudaMallocHost(&ws->h_asm, bytes_all));
        MPIC_CUDA(cudaMalloc(&ws->d_asm, bytes_all));
        ws->asm_cap = bytes_all;
    }
    if (!ap.chunks.empty()) std::memcpy(ws->h_asm, ap.chunks.data(), ap.chunks.size() * sizeof(AsmChunk));
    if (!ap.tables.empty())
        std::memcpy((char*)ws->h_asm + bytes_c, ap.tables.data(), ap.tables.size() * sizeof(float2));
    const AttnLink* d_link = nullptr;
    const uint8_t* d_skip = nullptr;
    if (link) {
        AttnLink* hl = reinterpret_cast<AttnLink*>((char*)ws->h_asm + off_l);
        std::memset(hl, 0, sizeof(AttnLink));
        make_link_maps(hl, ks.data(), vs.data(), ts.data(), n_img, linked->L, linked->H * linked->D);
        hl->nblk = (uint32_t)link_blk.size();
        std::memcpy(hl + 1, link_blk.data(), link_blk.size() * 4);
        std::memcpy(reinterpret_cast<uint32_t*>(hl + 1) + link_blk.size(), link_wtile.data(), link_wtile.size() * 2);
        std::memcpy((char*)ws->h_asm + off_s, link_skip.data(), link_skip.size());
        d_link = reinterpret_cast<const AttnLink*>((char*)ws->d_asm + off_l);
        d_skip = reinterpret_cast<const uint8_t*>((char*)ws->d_asm + off_s);
    }

    // ---- device work: one stream-ordered sequence, optionally recorded as a CUDA graph ----
    static const bool asm_overlap = [] {
        const char* e = getenv("MPIC_ASM_OVERLAP");  // diagnostics: 0 = assemble all layers up front
        return !e || atoi(e) != 0;
    }();
    auto enqueue = [&] {
        MPIC_CUDA(cudaMemcpyAsync(ws->d_ids, ws->h_ids, r.m * 4, cudaMemcpyHostToDevice, s));
        MPIC_CUDA(cudaMemcpyAsync(ws->d_rows, ws->h_rows, r.m * 4, cudaMemcpyHostToDevice, s));
        MPIC_CUDA(cudaMemcpyAsync(ws->d_asm, ws->h_asm, bytes_all, cudaMemcpyHostToDevice, s));
        const AsmChunk* dch = static_cast<const AsmChunk*>(ws->d_asm);
        const float2* dtab = reinterpret_cast<const float2*>((char*)ws->d_asm + bytes_c);
        std::function<void(uint32_t)> wait_layer;
        // per-layer overlap pays only when the copy is long enough to hide behind the GEMMs:
        // a large request whose chunks are NOT linked inside attention. With linking the
        // assembly is only the partial blocks (config C: 0.23 ms in one launch up front, the
        // same request time as overlapped); small requests assemble up front too (config B)
        uint64_t asm_bytes = 0;
        for (uint32_t i = 0; i < n_img; ++i)
            asm_bytes += (uint64_t)r.refs[i].rows * linked->L * linked->H * linked->D * esz(linked->dtype) * 2;
        if (asm_overlap && !link && asm_bytes >= (2ull << 30)) {
            // Layer l of the assembly runs on a side stream and only layer l's QKV waits for it:
            // the HBM-bound copy of layers l+1.. overlaps the tensor-bound GEMMs of layer l.
            ensure_asm_stream(ws, model->cfg.n_layers);
            const size_t plane = (size_t)linked->T * linked->H * linked->D * esz(linked->dtype);
            MPIC_CUDA(cudaEventRecord(ws->ev_asm_in, s));
            MPIC_CUDA(cudaStreamWaitEvent(ws->asm_stream, ws->ev_asm_in, 0));
            for (uint32_t l = 0; l < linked->L; ++l) {
                {
                    ProfScope ps(ws->asm_stream, MPIC_PHASE_ASSEMBLE);
                    launch_assemble(dch, n_img, dtab, ap.n_tables, src_t, (char*)linked->k + l * plane,
                                    (char*)linked->v + l * plane, linked->dtype, 1, linked->T, linked->H, linked->D, 1,
                                    ws->asm_stream, l, d_skip);
                }
                MPIC_CUDA(cudaEventRecord(ws->ev_asm[l], ws->asm_stream));
            }
            wait_layer = [&](uint32_t l) { MPIC_CUDA(cudaStreamWaitEvent(s, ws->ev_asm[l], 0)); };
        } else {
            ProfScope ps(s, MPIC_PHASE_ASSEMBLE);
            launch_assemble(dch, n_img, dtab, ap.n_tables, src_t, linked->k, linked->v, linked->dtype, linked->L,
                            linked->T, linked->H, linked->D, 1, s, 0, d_skip);
        }
        forward_rows(model, ws, ws->d_ids, ws->d_rows, ws->d_rows, r.m, r.n - 1, linked, ws->d_logits, s, wait_layer,
                     r.sel.data(), nullptr, /*plan_ready=*/true, d_link);
        MPIC_CUDA(cudaMemcpyAsync(ws->h_logits, ws->d_logits, model->cfg.vocab_size * 4, cudaMemcpyDeviceToHost, s));
    };
    GraphSig sig;
    sig.model = model;
    sig.linked_k = linked->k;
    sig.linked_v = linked->v;
    sig.rope = model->rope;
    sig.ws_gen = ws->gen;
    sig.n = r.n;
    sig.m = r.m;
    sig.n_img = n_img;
    sig.n_tables = ap.n_tables;
    sig.n_units = ws->n_units;
    sig.n_comb = ws->n_comb;
    sig.reposition = reposition;
    sig.src_dtype = src_t;
    sig.link = link;
    bool prof;
    {
        std::lock_guard<std::mutex> lk(g_prof_mu);
        prof = g_prof_on;
    }
    // the legacy default stream cannot be captured (the library is not built with
    // per-thread default streams): such requests always run eagerly
    const bool use_graph = ws->graphs && !prof && s != nullptr && s != cudaStreamLegacy;
    if (use_graph && ws->graph && ws->graph_sig == sig) {
        MPIC_CUDA(cudaGraphLaunch(ws->graph, s));
        note_launch(ws->graph_kernels);
    } else if (use_graph && ws->last_sig == sig) {
        // second request of this shape: record it once, replay it from now on
        if (ws->graph) {
            cudaGraphExecDestroy(ws->graph);
            ws->graph = nullptr;
        }
        const uint32_t before = g_launches;
        cudaGraph_t g = nullptr;
        MPIC_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
        try {
            enqueue();
        } catch (...) {
            cudaStreamEndCapture(s, &g);
            if (g) cudaGraphDestroy(g);
            throw;
        }
        MPIC_CUDA(cudaStreamEndCapture(s, &g));
        const cudaError_t ie = cudaGraphInstantiate(&ws->graph, g, 0);
        cudaGraphDestroy(g);
        MPIC_CUDA(ie);
        ws->graph_kernels = g_launches - before;
        ws->graph_sig = sig;
        MPIC_CUDA(cudaGraphLaunch(ws->graph, s));
    } else {
        enqueue();
    }
    ws->last_sig = sig;
    MPIC_CUDA(cudaStreamSynchronize(s));
    std::memcpy(logits, ws->h_logits, model->cfg.vocab_size * sizeof(float));
    if (selected) std::memcpy(selected, r.sel.data(), r.m * sizeof(uint32_t));
    if (m_out) *m_out = r.m;
    API_END
}

// ---- batched varlen requests (SURVEY §8b "a batched varlen variant") -------------------
// nreq independent requests in ONE selective pass: request r's cache occupies rows
// [off_r, off_r + n_r) of `linked` (off_r = sum of the earlier n), its selected rows are
// scattered there at their own positions (RoPE at the position, KV row = off_r + position),
// and attention masks every key outside [off_r, off_r + position]. The projections then see
// sum(m_r) rows at once instead of streaming every weight once per request.
int mpic_request_prefill_batch(mpic_model_t model, mpic_workspace_t ws, const mpic_prompt* prompts, uint32_t nreq,
                               const mpic_policy* policy, const mpic_kv_t* chunks, mpic_reposition reposition,
                               mpic_kv_t linked, float* logits, uint32_t* m_out, void* stream) {
    API_BEGIN
    MPIC_CUDA(cudaSetDevice(model->device));
    cudaStream_t s = (cudaStream_t)stream;
    MPIC_REQUIRE(ws && ws->model == model, MPIC_ERR_VALIDATION, "workspace belongs to another model");
    MPIC_REQUIRE(nreq > 0 && prompts && logits, MPIC_ERR_VALIDATION, "empty request batch");
    MPIC_REQUIRE(use_tc_attention(model), MPIC_ERR_VALIDATION,
                 "batched requests run on the bf16 head_dim-128 tensor-core path");
    const mpic_model_config& c = model->cfg;
    std::vector<RequestPlan> plans;
    plans.reserve(nreq);
    uint32_t n_tot = 0, m_tot = 0;
    for (uint32_t r = 0; r < nreq; ++r) {
        plans.push_back(plan_request(model, &prompts[r], policy, nullptr));
        n_tot += plans.back().n;
        m_tot += plans.back().m;
    }
    MPIC_REQUIRE(linked && linked->L == c.n_layers && linked->H == c.n_heads && linked->D == c.head_dim &&
                     linked->dtype == model->dtype,
                 MPIC_ERR_VALIDATION, "linked cache shape does not match model");
    MPIC_REQUIRE(linked->T >= n_tot, MPIC_ERR_CONTRACT, "linked cache shorter than the batch's prompts");
    MPIC_REQUIRE(m_tot <= ws->max_rows, MPIC_ERR_VALIDATION, "more rows than the workspace holds");
    std::vector<uint32_t> rows(m_tot), pos(m_tot), starts(m_tot), last(nreq);
    std::vector<int32_t> ids(m_tot);
    std::vector<mpic_chunk_ref> refs;
    std::vector<const void*> ks, vs;
    std::vector<uint32_t> ts;
    uint32_t off = 0, at = 0, ci = 0, max_pos = 0;
    for (uint32_t r = 0; r < nreq; ++r) {
        const RequestPlan& p = plans[r];
        check_ids(model, p.ids_sel.data(), p.m);
        for (uint32_t i = 0; i < p.m; ++i) {
            rows[at + i] = off + p.sel[i];
            pos[at + i] = p.sel[i];
            starts[at + i] = off;
            ids[at + i] = p.ids_sel[i];
            max_pos = std::max(max_pos, p.sel[i]);
        }
        for (mpic_chunk_ref ref : p.refs) {
            const mpic_kv_t ch = chunks[ci++];
            MPIC_REQUIRE(ch, MPIC_ERR_LINK, "no fetched entry for image segment");
            MPIC_REQUIRE(ch->T == ref.rows, MPIC_ERR_LINK, "token_count mismatch for image segment");
            MPIC_REQUIRE(ch->L == linked->L && ch->H == linked->H && ch->D == linked->D, MPIC_ERR_LINK,
                         "entry tensor shape does not match model");
            MPIC_REQUIRE(ch->dtype == chunks[0]->dtype, MPIC_ERR_VALIDATION, "mixed chunk dtypes");
            ref.dst_row0 += off;
            ref.position_base += off;  // Rerotate's delta (dst - base) stays request-relative
            refs.push_back(ref);
            ks.push_back(ch->k);
            vs.push_back(ch->v);
            ts.push_back(ch->T);
        }
        last[r] = at + p.m - 1;
        if (m_out) m_out[r] = p.m;
        at += p.m;
        off += p.n;
    }
    const uint32_t n_img = (uint32_t)refs.size();
    const mpic_dtype src_t = n_img ? chunks[0]->dtype : model->dtype;
    const AsmPlan ap = plan_assembly(ks.data(), vs.data(), ts.data(), refs.data(), n_img, linked->T, linked->D,
                                     reposition, c.rope_base, linked->H * linked->D);
    ensure_rope(model, max_pos + 1, s);
    prepare_attn_plan(ws, rows.data(), m_tot, n_tot - 1, c.n_heads, starts.data());
    const size_t bytes_c = std::max<size_t>(1, ap.chunks.size()) * sizeof(AsmChunk);
    const size_t bytes_t = std::max<size_t>(1, ap.tables.size()) * sizeof(float2);
    if (ws->asm_cap < bytes_c + bytes_t) {
        ++ws->gen;
        MPIC_CUDA(cudaDeviceSynchronize());
        cudaFreeHost(ws->h_asm);
        cudaFree(ws->d_asm);
        ws->h_asm = ws->d_asm = nullptr;
        ws->asm_cap = 0;
        MPIC_CUDA(cudaMallocHost(&ws->h_asm, bytes_c + bytes_t));
        MPIC_CUDA(cudaMalloc(&ws->d_asm, bytes_c + bytes_t));
        ws->asm_cap = bytes_c + bytes_t;
    }
    if (!ap.chunks.empty()) std::memcpy(ws->h_asm, ap.chunks.data(), ap.chunks.size() * sizeof(AsmChunk));
    if (!ap.tables.empty())
        std::memcpy((char*)ws->h_asm + bytes_c, ap.tables.data(), ap.tables.size() * sizeof(float2));
    std::memcpy(ws->h_ids, ids.data(), m_tot * 4);
    std::memcpy(ws->h_rows, rows.data(), m_tot * 4);
    std::memcpy(ws->h_pos, pos.data(), m_tot * 4);
    std::memcpy(ws->h_start, starts.data(), m_tot * 4);
    MPIC_CUDA(cudaMemcpyAsync(ws->d_ids, ws->h_ids, m_tot * 4, cudaMemcpyHostToDevice, s));
    MPIC_CUDA(cudaMemcpyAsync(ws->d_rows, ws->h_rows, m_tot * 4, cudaMemcpyHostToDevice, s));
    MPIC_CUDA(cudaMemcpyAsync(ws->d_pos, ws->h_pos, m_tot * 4, cudaMemcpyHostToDevice, s));
    MPIC_CUDA(cudaMemcpyAsync(ws->d_start, ws->h_start, m_tot * 4, cudaMemcpyHostToDevice, s));
    MPIC_CUDA(cudaMemcpyAsync(ws->d_asm, ws->h_asm, bytes_c + bytes_t, cudaMemcpyHostToDevice, s));
    {
        ProfScope ps(s, MPIC_PHASE_ASSEMBLE);
        launch_assemble(static_cast<const AsmChunk*>(ws->d_asm), n_img,
                        reinterpret_cast<const float2*>((char*)ws->d_asm + bytes_c), ap.n_tables, src_t, linked->k,
                        linked->v, linked->dtype, linked->L, linked->T, linked->H, linked->D, 1, s);
    }
    float* d_lg = nullptr;
    MPIC_CUDA(cudaMallocAsync((void**)&d_lg, (size_t)nreq * c.vocab_size * 4, s));
    forward_rows(model, ws, ws->d_ids, ws->d_rows, ws->d_pos, m_tot, max_pos, linked, d_lg, s, {}, rows.data(),
                 nullptr, /*plan_ready=*/true, nullptr, ws->d_start, &last);
    MPIC_CUDA(cudaMemcpyAsync(logits, d_lg, (size_t)nreq * c.vocab_size * 4, cudaMemcpyDeviceToHost, s));
    MPIC_CUDA(cudaFreeAsync(d_lg, s));
    MPIC_CUDA(cudaStreamSynchronize(s));
    API_END
}

// ---- head-parallel request ---------------------------------------------
// Rank r of P owns heads [r*H/P, (r+1)*H/P): its model holds those heads' Wq/Wk/Wv rows
// and the matching Wo columns (bit-identical slices of the synthetic weights) plus the full
// FFN; its request cache holds only its heads. Per layer: mpic_hp_layer_attn (QKV, attention,
// Wo partial sums of all h outputs) -> reduce-scatter of the partials across ranks (caller,
// NCCL) -> mpic_hp_layer_ffn on this rank's rows -> all-gather of the bf16 rows (caller).
int mpic_model_create_heads(const mpic_model_config* cfg, int device, mpic_dtype dtype, uint32_t head0,
                            uint32_t n_local_heads, mpic_model_t* out) {
    mpic_model_t m = nullptr;
    API_BEGIN
    validate_cfg(cfg);
    validate_device_cfg(cfg);
    MPIC_REQUIRE(n_local_heads > 0 && head0 + n_local_heads <= cfg->n_heads, MPIC_ERR_VALIDATION,
                 "head slice outside the model");
    set_device(device);
    m = new mpic_model_s();
    m->cfg = *cfg;
    m->device = device;
    m->dtype = dtype;
    m->head0 = head0;
    m->n_local_heads = n_local_heads;
    const size_t h = cfg->hidden_dim, V = cfg->vocab_size, L = cfg->n_layers, D = cfg->head_dim;
    const size_t hs = n_local_heads * D, e = esz(dtype);
    m->emb = dmalloc<float>(V * h);
    MPIC_CUDA(cudaMalloc(&m->lm_head, V * h * e));
    for (size_t l = 0; l < L; ++l) {
        void* p;
        MPIC_CUDA(cudaMalloc(&p, 3 * hs * h * e));
        m->wqkv.push_back(p);
        MPIC_CUDA(cudaMalloc(&p, h * hs * e));
        m->wo.push_back(p);
        MPIC_CUDA(cudaMalloc(&p, 4 * h * h * e));
        m->w1.push_back(p);
        MPIC_CUDA(cudaMalloc(&p, 4 * h * h * e));
        m->w2.push_back(p);
    }
    std::vector<double> inv(D / 2);
    for (uint32_t i = 0; i + 1 < D; i += 2)  // model.cpp:51-53
        inv[i / 2] = std::pow(static_cast<double>(cfg->rope_base), -static_cast<double>(i) / D);
    m->inv_freq = dmalloc<double>(D / 2);
    MPIC_CUDA(cudaMemcpy(m->inv_freq, inv.data(), inv.size() * sizeof(double), cudaMemcpyHostToDevice));
    const float scale = 1.0f / std::sqrt(static_cast<float>(h));  // model.cpp:106
    cudaStream_t s = 0;
    const uint32_t r0 = head0 * (uint32_t)D;
    launch_synth(cfg->seed, 100, 0, V * h, 1.0f, m->emb, MPIC_F32, s);
    launch_synth(cfg->seed, 101, 0, V * h, scale, m->lm_head, dtype, s);
    for (uint32_t l = 0; l < cfg->n_layers; ++l) {
        for (uint32_t part = 0; part < 3; ++part)  // rows [r0, r0+hs) of Wq, Wk, Wv
            launch_synth_2d(cfg->seed, 1 + part, l, (uint32_t)hs, (uint32_t)h, r0, 0, (uint32_t)h, scale,
                            (char*)m->wqkv[l] + part * hs * h * e, dtype, s);
        launch_synth_2d(cfg->seed, 4, l, (uint32_t)h, (uint32_t)h, 0, r0, (uint32_t)hs, scale, m->wo[l], dtype, s);
        launch_synth(cfg->seed, 5, l, 4 * h * h, scale, m->w1[l], dtype, s);
        launch_synth(cfg->seed, 6, l, 4 * h * h, scale, m->w2[l], dtype, s);
    }
    ensure_rope(m, 1, s);
    MPIC_CUDA(cudaDeviceSynchronize());
    *out = m;
    m = nullptr;
    API_END
}

int mpic_hp_prepare(mpic_model_t model, mpic_workspace_t ws, const mpic_prompt* prompt, const mpic_policy* policy,
                    const mpic_kv_t* chunks, mpic_reposition reposition, const uint32_t* position_bases,
                    mpic_kv_t linked, uint32_t* selected, uint32_t* m_out, void* stream) {
    API_BEGIN
    MPIC_CUDA(cudaSetDevice(model->device));
    cudaStream_t s = (cudaStream_t)stream;
    MPIC_REQUIRE(ws && ws->model == model, MPIC_ERR_VALIDATION, "workspace belongs to another model");
    MPIC_REQUIRE(model->n_local_heads && model->dtype == MPIC_BF16, MPIC_ERR_VALIDATION,
                 "head-parallel needs a bf16 head-slice model (mpic_model_create_heads)");
    const uint32_t D = model->cfg.head_dim, hs = model->n_local_heads * D, h = model->cfg.hidden_dim;
    const RequestPlan r = plan_request(model, prompt, policy, position_bases);
    MPIC_REQUIRE(linked && linked->L == model->cfg.n_layers && linked->T == r.n && linked->H == model->n_local_heads &&
                     linked->D == D && linked->dtype == model->dtype,
                 MPIC_ERR_VALIDATION, "request cache must be [L][n][local heads][D] of the model dtype");
    MPIC_REQUIRE(r.m <= ws->max_rows, MPIC_ERR_VALIDATION, "more rows than the workspace holds");
    check_ids(model, r.ids_sel.data(), r.m);
    const uint32_t n_img = (uint32_t)r.refs.size();
    std::vector<const void*> ks(n_img), vs(n_img);
    std::vector<uint32_t> ts(n_img);
    for (uint32_t i = 0; i < n_img; ++i) {
        const mpic_kv_t c = chunks[i];
        MPIC_REQUIRE(c, MPIC_ERR_LINK, "no fetched entry for image segment");
        MPIC_REQUIRE(c->T == r.refs[i].rows, MPIC_ERR_LINK, "token_count mismatch for image segment");
        MPIC_REQUIRE(c->L == linked->L && c->H == model->cfg.n_heads && c->D == D, MPIC_ERR_LINK,
                     "entry tensor shape does not match model");
        MPIC_REQUIRE(c->dtype == chunks[0]->dtype, MPIC_ERR_VALIDATION, "mixed chunk dtypes");
        ks[i] = c->k;
        vs[i] = c->v;
        ts[i] = c->T;
    }
    // this rank's head columns of every chunk -> its request cache
    const AsmPlan ap = plan_assembly(ks.data(), vs.data(), ts.data(), r.refs.data(), n_img, linked->T, D, reposition,
                                     model->cfg.rope_base, hs, h, model->head0 * D);
    const AsmChunk* dc;
    const float2* dt;
    void* buf = upload_plan(ap, s, &dc, &dt);
    {
        ProfScope ps(s, MPIC_PHASE_ASSEMBLE);
        launch_assemble(dc, n_img, dt, ap.n_tables, n_img ? chunks[0]->dtype : model->dtype, linked->k, linked->v,
                        linked->dtype, linked->L, linked->T, linked->H, D, 1, s);
    }
    MPIC_CUDA(cudaFreeAsync(buf, s));
    ensure_rope(model, r.n, s);
    std::memcpy(ws->h_ids, r.ids_sel.data(), r.m * sizeof(int32_t));
    std::memcpy(ws->h_rows, r.sel.data(), r.m * sizeof(uint32_t));
    MPIC_CUDA(cudaMemcpyAsync(ws->d_ids, ws->h_ids, r.m * 4, cudaMemcpyHostToDevice, s));
    MPIC_CUDA(cudaMemcpyAsync(ws->d_rows, ws->h_rows, r.m * 4, cudaMemcpyHostToDevice, s));
    MPIC_CUDA(cudaMemsetAsync(ws->x, 0, (size_t)ws->m_pad * h * sizeof(float), s));
    MPIC_CUDA(cudaMemsetAsync(ws->xb, 0, (size_t)ws->m_pad * h * 2, s));
    {
        ProfScope ps(s, MPIC_PHASE_EMBED);
        launch_embed(model->emb, ws->d_ids, r.m, h, ws->x, ws->xb, s);
    }
    launch_rope_gather(model->rope, ws->d_rows, r.m, D / 2, ws->rope_tok, s);
    if (use_tc_attention(model)) {
        prepare_attn_plan(ws, r.sel.data(), r.m, r.n - 1, model->n_local_heads);
        enqueue_attn_plan(ws, s);
    }
    ws->hp_m = r.m;
    ws->hp_n = r.n;
    if (selected) std::memcpy(selected, r.sel.data(), r.m * sizeof(uint32_t));
    if (m_out) *m_out = r.m;
    API_END
}

}  // extern "C"

namespace {
// One layer of a head-parallel rank (see mpic_hp_layer_attn / mpic_hp_layer_ffn).
void hp_attn(mpic_model_t md, mpic_workspace_t ws, uint32_t l, mpic_kv_t kv, float* d_partial, cudaStream_t s) {
    MPIC_REQUIRE(md->n_local_heads && ws->hp_m && l < md->cfg.n_layers, MPIC_ERR_STATE,
                 "mpic_hp_prepare must run first");
    const uint32_t m = ws->hp_m, h = md->cfg.hidden_dim, D = md->cfg.head_dim, Hl = md->n_local_heads,
                   hs = Hl * D;
    const size_t plane = (size_t)kv->T * hs * 2;
    void* kl = (char*)kv->k + l * plane;
    void* vl = (char*)kv->v + l * plane;
    EpiParams qkv;
    qkv.mode = EPI_QKV;
    qkv.q = ws->q;
    qkv.kv_k = kl;
    qkv.kv_v = vl;
    qkv.kv_rows = ws->d_rows;
    qkv.rope_pos = ws->d_rows;
    qkv.rope = md->rope;
    qkv.rope_tok = ws->rope_tok;
    qkv.hidden = hs;
    qkv.head_dim = D;
    {
        ProfScope ps(s, MPIC_PHASE_QKV);
        run_gemm(md, ws->xb, md->wqkv[l], m, 3 * hs, h, qkv, s);
    }
    {
        ProfScope ps(s, MPIC_PHASE_ATTN);
        MPIC_REQUIRE(use_tc_attention(md), MPIC_ERR_VALIDATION, "head-parallel attention needs head_dim 128");
        launch_attn_tc(static_cast<const __nv_bfloat16*>(ws->q), static_cast<const __nv_bfloat16*>(kl),
                       static_cast<const __nv_bfloat16*>(vl), kv->T, ws->d_rows, m, Hl, ws->d_units, ws->n_units,
                       ws->d_comb, ws->n_comb, ws->part_o, ws->part_ml, static_cast<__nv_bfloat16*>(ws->attn), s,
                       nullptr, 0, nullptr, fused_combine() ? ws->d_comb_cnt : nullptr);
    }
    EpiParams st;
    st.mode = EPI_STORE_F32;
    st.out = d_partial;
    st.ldo = h;
    {
        ProfScope ps(s, MPIC_PHASE_WO);
        run_gemm(md, ws->attn, md->wo[l], m, h, hs, st, s);
    }
}

void hp_ffn(mpic_model_t md, mpic_workspace_t ws, uint32_t l, const float* d_reduced, uint32_t row0, uint32_t rows,
            cudaStream_t s) {
    MPIC_REQUIRE(md->n_local_heads && ws->hp_m && l < md->cfg.n_layers, MPIC_ERR_STATE,
                 "mpic_hp_prepare must run first");
    MPIC_REQUIRE(row0 + rows <= ws->m_pad, MPIC_ERR_VALIDATION, "row range outside the workspace");
    if (rows == 0) return;
    const uint32_t h = md->cfg.hidden_dim;
    float* x = ws->x + (size_t)row0 * h;
    __nv_bfloat16* xb = ws->xb + (size_t)row0 * h;
    launch_resid_add(x, d_reduced, xb, (size_t)rows * h, s);  // x += sum of the ranks' Wo partials
    EpiParams gl;
    gl.mode = EPI_GELU;
    gl.out = ws->ffn;
    gl.ldo = 4 * h;
    {
        ProfScope ps(s, MPIC_PHASE_W1);
        run_gemm(md, xb, md->w1[l], rows, 4 * h, h, gl, s);
    }
    EpiParams res;
    res.mode = EPI_RESID;
    res.x = x;
    res.ldx = h;
    res.xb = xb;
    res.partial = ws->partial;
    res.partial_cap = ws->partial_cap;
    {
        ProfScope ps(s, MPIC_PHASE_W2);
        run_gemm(md, ws->ffn, md->w2[l], rows, h, 4 * h, res, s);
    }
}
}  // namespace

extern "C" {

int mpic_hp_layer_attn(mpic_model_t md, mpic_workspace_t ws, uint32_t l, mpic_kv_t kv, float* d_partial,
                       void* stream) {
    API_BEGIN
    MPIC_CUDA(cudaSetDevice(md->device));
    hp_attn(md, ws, l, kv, d_partial, (cudaStream_t)stream);
    API_END
}

int mpic_hp_layer_ffn(mpic_model_t md, mpic_workspace_t ws, uint32_t l, const float* d_reduced, uint32_t row0,
                      uint32_t rows, void* stream) {
    API_BEGIN
    MPIC_CUDA(cudaSetDevice(md->device));
    hp_ffn(md, ws, l, d_reduced, row0, rows, (cudaStream_t)stream);
    API_END
}

int mpic_hp_logits(mpic_model_t md, mpic_workspace_t ws, uint32_t row, float* logits, void* stream) {
    API_BEGIN
    MPIC_CUDA(cudaSetDevice(md->device));
    cudaStream_t s = (cudaStream_t)stream;
    MPIC_REQUIRE(row < ws->m_pad, MPIC_ERR_VALIDATION, "row outside the workspace");
    const uint32_t h = md->cfg.hidden_dim;
    {
        ProfScope ps(s, MPIC_PHASE_LM_HEAD);
        launch_lm_head(ws->x + (size_t)row * h, md->lm_head, md->dtype, md->cfg.vocab_size, h, ws->d_logits, s);
    }
    MPIC_CUDA(cudaMemcpyAsync(ws->h_logits, ws->d_logits, md->cfg.vocab_size * 4, cudaMemcpyDeviceToHost, s));
    MPIC_CUDA(cudaStreamSynchronize(s));
    std::memcpy(logits, ws->h_logits, md->cfg.vocab_size * sizeof(float));
    API_END
}

// ---- head-parallel request inside the library, collectives over NCCL -----
// NCCL is resolved at run time (dlopen of libnccl.so.2: the process's copy when torch has
// already loaded one, else the system library), so the library itself carries no link-time
// NCCL dependency and every non-head-parallel entry point works without it.
}  // extern "C"

namespace {
struct NcclApi {
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    ncclResult_t (*comm_count)(const ncclComm_t, int*) = nullptr;
    ncclResult_t (*comm_user_rank)(const ncclComm_t, int*) = nullptr;
    ncclResult_t (*reduce_scatter)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                                   cudaStream_t) = nullptr;
    ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
    std::string why;
};

const NcclApi& nccl() {
    static const NcclApi api = [] {
        NcclApi a;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            const char* e = dlerror();
            a.why = std::string("cannot load libnccl.so.2: ") + (e ? e : "?");
            return a;
        }
        auto sym = [&](auto& fn, const char* name) {
            fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
            if (!fn && a.why.empty()) a.why = std::string("libnccl.so.2 lacks ") + name;
        };
        sym(a.get_unique_id, "ncclGetUniqueId");
        sym(a.comm_init_rank, "ncclCommInitRank");
        sym(a.comm_destroy, "ncclCommDestroy");
        sym(a.comm_count, "ncclCommCount");
        sym(a.comm_user_rank, "ncclCommUserRank");
        sym(a.reduce_scatter, "ncclReduceScatter");
        sym(a.all_gather, "ncclAllGather");
        sym(a.broadcast, "ncclBroadcast");
        sym(a.error_string, "ncclGetErrorString");
        return a;
    }();
    MPIC_REQUIRE(api.why.empty(), MPIC_ERR_STATE, api.why);
    return api;
}

#define MPIC_NCCL(call)                                                                          \
    do {                                                                                         \
        const ncclResult_t r_ = (call);                                                          \
        if (r_ != ncclSuccess)                                                                   \
            throw Error(MPIC_ERR_CUDA, std::string("NCCL: ") + #call + ": " + nccl().error_string(r_)); \
    } while (0)

// Grow a device buffer to `need` floats (contents undefined), bumping the workspace
// generation so a recorded layer-loop graph is not replayed on freed memory.
void grow_f32(mpic_workspace_t ws, float*& p, size_t& cap, size_t need) {
    if (cap >= need) return;
    MPIC_CUDA(cudaDeviceSynchronize());
    cudaFree(p);
    p = nullptr;
    MPIC_CUDA(cudaMalloc(&p, std::max<size_t>(need, 1) * sizeof(float)));
    cap = need;
    ++ws->gen;
}
}  // namespace

extern "C" {

int mpic_nccl_unique_id(uint8_t* out) {
    API_BEGIN
    MPIC_REQUIRE(out, MPIC_ERR_VALIDATION, "null argument");
    static_assert(sizeof(ncclUniqueId) == MPIC_NCCL_ID_BYTES, "ncclUniqueId size");
    ncclUniqueId id;
    MPIC_NCCL(nccl().get_unique_id(&id));
    std::memcpy(out, &id, sizeof(id));
    API_END
}

int mpic_nccl_comm_create(const uint8_t* id, int nranks, int rank, int device, void** out) {
    API_BEGIN
    MPIC_REQUIRE(id && out && nranks > 0 && rank >= 0 && rank < nranks, MPIC_ERR_VALIDATION, "bad communicator request");
    set_device(device);
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    ncclComm_t c = nullptr;
    MPIC_NCCL(nccl().comm_init_rank(&c, nranks, uid, rank));
    *out = c;
    API_END
}

int mpic_nccl_comm_destroy(void* comm) {
    API_BEGIN
    if (comm) MPIC_NCCL(nccl().comm_destroy(static_cast<ncclComm_t>(comm)));
    API_END
}

int mpic_hp_request(mpic_model_t md, mpic_workspace_t ws, void* comm, const mpic_prompt* prompt,
                    const mpic_policy* policy, const mpic_kv_t* chunks, mpic_reposition reposition,
                    const uint32_t* position_bases, mpic_kv_t linked, float* logits, uint32_t* selected,
                    uint32_t* m_out, void* stream) {
    API_BEGIN
    MPIC_CUDA(cudaSetDevice(md->device));
    cudaStream_t s = (cudaStream_t)stream;
    ncclComm_t c = static_cast<ncclComm_t>(comm);
    int P = 1, rank = 0;
    if (c) {
        MPIC_NCCL(nccl().comm_count(c, &P));
        MPIC_NCCL(nccl().comm_user_rank(c, &rank));
    }
    const uint32_t H = md->cfg.n_heads, h = md->cfg.hidden_dim, L = md->cfg.n_layers, V = md->cfg.vocab_size;
    MPIC_REQUIRE(md->n_local_heads && md->n_local_heads * (uint32_t)P == H &&
                     md->head0 == (uint32_t)rank * md->n_local_heads,
                 MPIC_ERR_VALIDATION, "the model must hold heads [rank*H/P, (rank+1)*H/P) of the communicator rank");
    // step 0: this rank's head slice of the request cache, embeddings, plans
    uint32_t m = 0;
    {
        const uint32_t launches = g_launches;
        const int rc = mpic_hp_prepare(md, ws, prompt, policy, chunks, reposition, position_bases, linked, selected,
                                       &m, stream);
        g_launches += launches;
        if (rc != MPIC_OK) throw Error(rc, g_last_error);
    }
    const uint32_t mr = ceil_div(m, (uint32_t)P), m_pad = mr * (uint32_t)P;
    MPIC_REQUIRE(m_pad <= ws->m_pad, MPIC_ERR_VALIDATION,
                 "P * ceil(m / P) rows exceed the workspace: create it with max_rows >= m + P");
    grow_f32(ws, ws->hp_partial, ws->hp_partial_cap, (size_t)m_pad * h);
    grow_f32(ws, ws->hp_reduced, ws->hp_reduced_cap, (size_t)mr * h);
    // partial rows >= m are never written by the Wo GEMM: they must be zero for the reduction
    if (m_pad > m) MPIC_CUDA(cudaMemsetAsync(ws->hp_partial + (size_t)m * h, 0, (size_t)(m_pad - m) * h * 4, s));
    const uint32_t owner = (m - 1) / mr;
    auto layers = [&] {
        for (uint32_t l = 0; l < L; ++l) {
            hp_attn(md, ws, l, linked, ws->hp_partial, s);  // QKV + attention of my heads, my share of attn.Wo^T
            if (c) MPIC_NCCL(nccl().reduce_scatter(ws->hp_partial, ws->hp_reduced, (size_t)mr * h, ncclFloat32, ncclSum, c, s));
            else MPIC_CUDA(cudaMemcpyAsync(ws->hp_reduced, ws->hp_partial, (size_t)mr * h * 4, cudaMemcpyDeviceToDevice, s));
            hp_ffn(md, ws, l, ws->hp_reduced, (uint32_t)rank * mr, mr, s);  // residual + FFN on my rows
            if (c)  // in place: my rows are already at their offset of xb
                MPIC_NCCL(nccl().all_gather(ws->xb + (size_t)rank * mr * h, ws->xb, (size_t)mr * h, ncclBfloat16, c, s));
        }
        if ((uint32_t)rank == owner) {
            ProfScope ps(s, MPIC_PHASE_LM_HEAD);
            launch_lm_head(ws->x + (size_t)(m - 1) * h, md->lm_head, md->dtype, V, h, ws->d_logits, s);
        }
        if (c && P > 1) MPIC_NCCL(nccl().broadcast(ws->d_logits, ws->d_logits, V, ncclFloat32, (int)owner, c, s));
        MPIC_CUDA(cudaMemcpyAsync(ws->h_logits, ws->d_logits, V * 4, cudaMemcpyDeviceToHost, s));
    };
    // CUDA-graph replay of the layer loop (kernels + collectives): same key = same launches
    uint64_t key = 0xcbf29ce484222325ull;
    for (uint64_t v : {(uint64_t)(uintptr_t)md, (uint64_t)(uintptr_t)c, (uint64_t)(uintptr_t)linked->k,
                       (uint64_t)(uintptr_t)linked->v, (uint64_t)(uintptr_t)md->rope, ws->gen, (uint64_t)m,
                       (uint64_t)linked->T, (uint64_t)ws->n_units, (uint64_t)ws->n_comb})
        key = (key ^ v) * 0x100000001b3ull;
    bool prof;
    {
        std::lock_guard<std::mutex> lk(g_prof_mu);
        prof = g_prof_on;
    }
    const bool use_graph = ws->graphs && !prof && s != nullptr && s != cudaStreamLegacy;
    if (use_graph && ws->hp_graph && ws->hp_graph_key == key) {
        MPIC_CUDA(cudaGraphLaunch(ws->hp_graph, s));
        note_launch(ws->hp_graph_kernels);
    } else if (use_graph && ws->hp_last_key == key) {
        if (ws->hp_graph) {
            cudaGraphExecDestroy(ws->hp_graph);
            ws->hp_graph = nullptr;
        }
        const uint32_t before = g_launches;
        cudaGraph_t g = nullptr;
        MPIC_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
        try {
            layers();
        } catch (...) {
            cudaStreamEndCapture(s, &g);
            if (g) cudaGraphDestroy(g);
            throw;
        }
        MPIC_CUDA(cudaStreamEndCapture(s, &g));
        const cudaError_t ie = cudaGraphInstantiate(&ws->hp_graph, g, 0);
        cudaGraphDestroy(g);
        MPIC_CUDA(ie);
        ws->hp_graph_kernels = g_launches - before;
        ws->hp_graph_key = key;
        MPIC_CUDA(cudaGraphLaunch(ws->hp_graph, s));
    } else {
        layers();
    }
    ws->hp_last_key = key;
    MPIC_CUDA(cudaStreamSynchronize(s));
    std::memcpy(logits, ws->h_logits, V * sizeof(float));
    if (m_out) *m_out = m;
    API_END
}

int mpic_workspace_device_ptr(mpic_workspace_t ws, int which, void** out) {
    API_BEGIN
    MPIC_REQUIRE(ws && out, MPIC_ERR_VALIDATION, "null argument");
    switch (which) {
        case 0: *out = ws->x; break;    // residual stream fp32 [m_pad][h]
        case 1: *out = ws->xb; break;   // its bf16 copy [m_pad][h]
        default: throw Error(MPIC_ERR_VALIDATION, "unknown workspace buffer");
    }
    API_END
}

int mpic_workspace_set_graphs(mpic_workspace_t ws, int on) {
    API_BEGIN
    MPIC_REQUIRE(ws, MPIC_ERR_VALIDATION, "null workspace");
    ws->graphs = on != 0;
    if (!ws->graphs && ws->graph) {
        cudaGraphExecDestroy(ws->graph);
        ws->graph = nullptr;
    }
    API_END
}

int mpic_request_prefill_host2(mpic_model_t model, mpic_workspace_t ws, const mpic_prompt* prompt,
                               const mpic_policy* policy, const void* const* chunk_k, const void* const* chunk_v,
                               mpic_dtype chunk_dtype, const uint32_t* position_bases, mpic_reposition reposition,
                               mpic_kv_t linked, float* logits, uint32_t* selected, uint32_t* m_out, void* stream) {
    API_BEGIN
    const size_t es = esz(chunk_dtype);
    MPIC_CUDA(cudaSetDevice(model->device));
    cudaStream_t s = (cudaStream_t)stream;
    const RequestPlan r0 = plan_request(model, prompt, policy, nullptr);
    const uint32_t n_img = (uint32_t)r0.refs.size();
    // a NULL chunk is a miss: computed on the device at position base 0 (compute lane)
    std::vector<uint32_t> bases(n_img, 0);
    std::vector<bool> miss(n_img, false);
    for (uint32_t i = 0; i < n_img; ++i) {
        miss[i] = !chunk_k || !chunk_v || !chunk_k[i] || !chunk_v[i];
        if (!miss[i] && position_bases) bases[i] = position_bases[i];
    }
    const RequestPlan r = plan_request(model, prompt, policy, bases.data());
    check_linked(model, linked, r.n);
    const size_t h = model->cfg.hidden_dim;
    // Staging slot = one layer of every chunk in the Host tier's dtype, K then V.
    std::vector<size_t> off(n_img);
    size_t img_rows = 0;
    for (uint32_t i = 0; i < n_img; ++i) {
        off[i] = img_rows * h;
        img_rows += r.refs[i].rows;
    }
    const size_t slot_bytes = std::max<size_t>(1, img_rows) * h * es * 2;
    if (ws->stage_cap < slot_bytes) {
        MPIC_CUDA(cudaStreamSynchronize(ws->copy_stream));
        for (int i = 0; i < 2; ++i) {
            cudaFree(ws->stage[i]);
            ws->stage[i] = nullptr;
            MPIC_CUDA(cudaMalloc(&ws->stage[i], slot_bytes));
        }
        ws->stage_cap = slot_bytes;
    }
    // Per-slot placement plans (source pointers differ by slot; L = 1 per launch).
    std::vector<uint32_t> ts(n_img);
    for (uint32_t i = 0; i < n_img; ++i) ts[i] = r.refs[i].rows;
    const AsmChunk* dc[2];
    const float2* dt[2];
    void* bufs[2];
    uint32_t n_tab = 0;
    for (int sl = 0; sl < 2; ++sl) {
        std::vector<const void*> ks(n_img), vs(n_img);
        char* base = static_cast<char*>(ws->stage[sl]);
        for (uint32_t i = 0; i < n_img; ++i) {
            ks[i] = base + off[i] * es;
            vs[i] = base + (img_rows * h + off[i]) * es;
        }
        const AsmPlan p = plan_assembly(ks.data(), vs.data(), ts.data(), r.refs.data(), n_img,
                                        linked->T, linked->D, reposition, model->cfg.rope_base, linked->H * linked->D);
        n_tab = p.n_tables;
        bufs[sl] = upload_plan(p, s, &dc[sl], &dt[sl]);
    }
    const size_t e = esz(linked->dtype);
    const size_t plane = (size_t)linked->T * h * e;
    cudaStream_t cs = ws->copy_stream;
    MissLane lane(model, ws);
    {
        const std::vector<const uint8_t*> hashes = image_hashes(prompt);
        for (uint32_t i = 0; i < n_img; ++i)
            if (miss[i]) lane.start(i, hashes[i], r.refs[i].rows);
    }
    // The leading rows of a chunk that the request recomputes anyway (MPIC-k: its first k)
    // are not copied: the assembly moves whatever the staging slot holds there and the
    // layer's QKV scatter overwrites those cache rows before anything reads them.
    std::vector<uint32_t> lead(n_img, 0);
    for (uint32_t i = 0; i < n_img; ++i) {
        const uint32_t d0 = r.refs[i].dst_row0;
        auto it = std::lower_bound(r.sel.begin(), r.sel.end(), d0);
        while (it != r.sel.end() && lead[i] < r.refs[i].rows && *it == d0 + lead[i]) {
            ++lead[i];
            ++it;
        }
    }
    // The copy lane may not start before the plans (and any earlier user of the ring)
    // are done on the compute stream.
    MPIC_CUDA(cudaEventRecord(ws->ev_free[0], s));
    MPIC_CUDA(cudaEventRecord(ws->ev_free[1], s));
    auto issue_copy = [&](uint32_t l) {
        const int sl = l & 1;
        char* base = static_cast<char*>(ws->stage[sl]);
        MPIC_CUDA(cudaStreamWaitEvent(cs, ws->ev_free[sl], 0));
        for (uint32_t i = 0; i < n_img; ++i) {
            if (miss[i]) {
                lane.copy_layer(*lane.find(i), l, base + off[i] * es, base + (img_rows * h + off[i]) * es, chunk_dtype,
                                cs);
                continue;
            }
            const size_t cnt = (size_t)r.refs[i].rows * h, skip = (size_t)lead[i] * h;
            if (skip == cnt) continue;
            MPIC_CUDA(cudaMemcpyAsync(base + (off[i] + skip) * es,
                                      static_cast<const char*>(chunk_k[i]) + ((size_t)l * cnt + skip) * es,
                                      (cnt - skip) * es, cudaMemcpyHostToDevice, cs));
            MPIC_CUDA(cudaMemcpyAsync(base + (img_rows * h + off[i] + skip) * es,
                                      static_cast<const char*>(chunk_v[i]) + ((size_t)l * cnt + skip) * es,
                                      (cnt - skip) * es, cudaMemcpyHostToDevice, cs));
        }
        MPIC_CUDA(cudaEventRecord(ws->ev_ready[sl], cs));
    };
    const uint32_t L = model->cfg.n_layers;
    issue_copy(0);
    auto before_layer = [&](uint32_t l) {
        if (l + 1 < L) issue_copy(l + 1);  // waits for layer l-1's assembly to free the slot
        const int sl = l & 1;
        MPIC_CUDA(cudaStreamWaitEvent(s, ws->ev_ready[sl], 0));
        ProfScope ps(s, MPIC_PHASE_ASSEMBLE);
        launch_assemble(dc[sl], n_img, dt[sl], n_tab, chunk_dtype, (char*)linked->k + l * plane,
                        (char*)linked->v + l * plane, linked->dtype, 1, linked->T, linked->H,
                        linked->D, 1, s);
        MPIC_CUDA(cudaEventRecord(ws->ev_free[sl], s));
    };
    run_request(model, ws, r, linked, logits, selected, m_out, s, before_layer);
    for (int sl = 0; sl < 2; ++sl) MPIC_CUDA(cudaFreeAsync(bufs[sl], s));
    API_END
}

int mpic_request_prefill_host(mpic_model_t model, mpic_workspace_t ws, const mpic_prompt* prompt,
                              const mpic_policy* policy, const float* const* chunk_k,
                              const float* const* chunk_v, const uint32_t* position_bases,
                              mpic_reposition reposition, mpic_kv_t linked, float* logits,
                              uint32_t* selected, uint32_t* m_out, void* stream) {
    return mpic_request_prefill_host2(model, ws, prompt, policy, reinterpret_cast<const void* const*>(chunk_k),
                                      reinterpret_cast<const void* const*>(chunk_v), MPIC_F32, position_bases,
                                      reposition, linked, logits, selected, m_out, stream);
}

// ---- disk loader: .mpic files -> pinned ring -> HBM, overlapped with the layer loop ----
// The .mpic container (proj/src/cache.cpp:97-188): 84-byte header, K [L][T][h] then V
// [L][T][h] (v1: fp32, dtype 0; v2: bf16, dtype 1), then the zlib CRC32 of everything
// before it. v3 (this library's writer, mpic.write_mpic) adds a table of per-layer CRCs
// (crc_k[L], crc_v[L], each over that layer's segment alone) between the payload and the
// file CRC, so that every layer is verified BEFORE it is copied to the device.
//
// Reader threads pread layer l of every loaded chunk into a pinned slot laid out like the
// device staging slot and CRC each piece on the way; the copy stream moves the slot to HBM
// while layer l-1 computes. Fault semantics follow prepare (proj/src/transfer.cpp:83-145):
//   * a chunk whose file does not exist (or whose path is NULL) is a miss: computed;
//   * a file that cannot be used — wrong magic/version/size, another model's fingerprint,
//     wrong shape or token count, a content hash other than the prompt's image hash
//     (CacheStore::fetch, cache.cpp:171-176), a short read, a CRC mismatch — is a
//     fallback: computed instead;
// and computed chunks come from the compute lane (MissLane) concurrently with the loads.
// v3 layer CRCs are checked before the layer's H2D is issued: a mismatch aborts the pass
// and the request is re-run with that chunk computed. v1/v2 files carry only the file CRC,
// known once every layer has been read: a mismatch there also re-runs the request with the
// chunk computed, so the caller never receives logits or a linked cache built from a
// corrupt chunk.
namespace {
struct MpicFile {
    int fd = -1;
    uint32_t version = 0, position_base = 0, L = 0, T = 0, H = 0, D = 0;
    mpic_dtype dtype = MPIC_F32;
    uint64_t fingerprint = 0;
    uint32_t crc_stored = 0, crc_header = 0;
    std::vector<uint32_t> table;      // v3: crc_k[L] then crc_v[L]
    std::vector<uint32_t> crc_piece;  // [2][L][pieces] CRCs of the pieces as read
    std::vector<uint32_t> layer_crc;  // [2][L] per-layer CRCs computed on the GPU
    ~MpicFile() {
        if (fd >= 0) close(fd);
    }
};

void pread_all(int fd, void* dst, size_t n, off_t off) {
    char* p = static_cast<char*>(dst);
    while (n) {
        const ssize_t r = pread(fd, p, std::min<size_t>(n, (size_t)1 << 30), off);
        MPIC_REQUIRE(r > 0, MPIC_ERR_IO, "short read of a .mpic file");
        p += r;
        n -= (size_t)r;
        off += r;
    }
}

uint32_t crc_of(const void* p, size_t n) {
    uLong c = crc32(0L, Z_NULL, 0);
    const Bytef* b = static_cast<const Bytef*>(p);
    while (n) {
        const uInt c1 = (uInt)std::min<size_t>(n, (size_t)1 << 30);
        c = crc32(c, b, c1);
        b += c1;
        n -= c1;
    }
    return (uint32_t)c;
}

// Header checks of CacheStore::fetch / read_entry (cache.cpp:127-176, 261-304). Throws
// NOT_FOUND when the file does not exist, another class when it exists but is unusable.
void open_mpic(MpicFile& f, const char* path, const mpic_model_t md, uint32_t want_T, const uint8_t* want_hash) {
    f.fd = open(path, O_RDONLY);
    MPIC_REQUIRE(f.fd >= 0 || errno != ENOENT, MPIC_ERR_NOT_FOUND, std::string("no such chunk file: ") + path);
    MPIC_REQUIRE(f.fd >= 0, MPIC_ERR_IO, std::string("cannot open ") + path);
    struct stat st;
    MPIC_REQUIRE(fstat(f.fd, &st) == 0, MPIC_ERR_IO, "cannot stat a .mpic file");
    MPIC_REQUIRE(st.st_size >= 88, MPIC_ERR_FORMAT, ".mpic file too short");
    uint8_t h[84];
    pread_all(f.fd, h, sizeof(h), 0);
    auto u32 = [&](size_t o) { uint32_t v; std::memcpy(&v, h + o, 4); return v; };
    MPIC_REQUIRE(std::memcmp(h, "MPIC", 4) == 0, MPIC_ERR_FORMAT, "bad .mpic magic");
    f.version = u32(4);
    MPIC_REQUIRE(f.version >= 1 && f.version <= 3, MPIC_ERR_FORMAT, "unsupported .mpic version");
    std::memcpy(&f.fingerprint, h + 8, 8);
    f.position_base = u32(56);
    f.L = u32(60);
    f.T = u32(64);
    f.H = u32(68);
    f.D = u32(72);
    const uint8_t dt = h[76];
    MPIC_REQUIRE((f.version == 1 && dt == 0) || (f.version >= 2 && (dt == 0 || dt == 1)), MPIC_ERR_FORMAT,
                 "unsupported .mpic payload dtype");
    f.dtype = dt == 1 ? MPIC_BF16 : MPIC_F32;
    const mpic_model_config& c = md->cfg;
    MPIC_REQUIRE(f.fingerprint == fingerprint_of(&c), MPIC_ERR_LINK, "chunk was computed by a different model");
    MPIC_REQUIRE(std::memcmp(h + 24, want_hash, 32) == 0, MPIC_ERR_INTEGRITY, "content hash mismatch on load");
    MPIC_REQUIRE(f.L == c.n_layers && f.H == c.n_heads && f.D == c.head_dim, MPIC_ERR_LINK,
                 "entry tensor shape does not match model");
    MPIC_REQUIRE(f.T == want_T, MPIC_ERR_LINK, "token_count mismatch for image segment");
    const size_t payload = 2 * (size_t)f.L * f.T * f.H * f.D * esz(f.dtype);
    const size_t table = f.version == 3 ? 2 * (size_t)f.L * 4 : 0;
    const size_t want = 84 + payload + table + 4;
    MPIC_REQUIRE((size_t)st.st_size == want, MPIC_ERR_FORMAT, ".mpic file size does not match its header");
    if (table) {
        f.table.resize(2 * f.L);
        pread_all(f.fd, f.table.data(), table, (off_t)(84 + payload));
    }
    uint8_t tail[4];
    pread_all(f.fd, tail, 4, (off_t)(want - 4));
    std::memcpy(&f.crc_stored, tail, 4);
    f.crc_header = crc_of(h, sizeof(h));
}

// Thrown from the layer loop when a loaded chunk turns out to be unusable mid-request.
struct RerunWithCompute {
    uint32_t chunk;
};

// One pass of a files request with a fixed set of chunks to compute. Returns the chunk
// whose file failed verification (the caller re-runs with it computed), or -1 on success.
int files_pass(mpic_model_t model, mpic_workspace_t ws, const mpic_prompt* prompt, const mpic_policy* policy,
               const char* const* paths, mpic_reposition reposition, mpic_kv_t linked, float* logits,
               uint32_t* selected, uint32_t* m_out, cudaStream_t s, std::vector<uint32_t>& status,
               std::vector<std::unique_ptr<MpicFile>>& files) {
    const RequestPlan r0 = plan_request(model, prompt, policy, nullptr);
    const uint32_t n_img = (uint32_t)r0.refs.size();
    const std::vector<const uint8_t*> hashes = image_hashes(prompt);
    std::vector<uint32_t> bases(n_img, 0);
    for (uint32_t i = 0; i < n_img; ++i)
        if (status[i] == MPIC_CHUNK_LOADED) bases[i] = files[i]->position_base;
    const RequestPlan r = plan_request(model, prompt, policy, bases.data());
    mpic_dtype ct = model->dtype;  // slot dtype: the files' payload dtype, else the model's
    bool any_loaded = false;
    for (uint32_t i = 0; i < n_img; ++i)
        if (status[i] == MPIC_CHUNK_LOADED) {
            if (!any_loaded) ct = files[i]->dtype;
            MPIC_REQUIRE(files[i]->dtype == ct, MPIC_ERR_VALIDATION, "mixed chunk dtypes");
            any_loaded = true;
        }
    const size_t es = esz(ct), h = model->cfg.hidden_dim;
    const uint32_t L = model->cfg.n_layers;
    // slot layout: loaded chunks first (one contiguous H2D per K / V region), then computed
    std::vector<size_t> off(n_img);
    size_t img_rows = 0, loaded_rows = 0;
    for (int pass = 0; pass < 2; ++pass)
        for (uint32_t i = 0; i < n_img; ++i)
            if ((status[i] == MPIC_CHUNK_LOADED) == (pass == 0)) {
                off[i] = img_rows * h;
                img_rows += r.refs[i].rows;
                if (pass == 0) loaded_rows = img_rows;
            }
    const size_t slot_bytes = std::max<size_t>(1, img_rows) * h * es * 2;
    constexpr int kSlots = 3;
    if (ws->stage_cap < slot_bytes) {
        MPIC_CUDA(cudaDeviceSynchronize());
        for (int i = 0; i < 2; ++i) {
            cudaFree(ws->stage[i]);
            ws->stage[i] = nullptr;
            MPIC_CUDA(cudaMalloc(&ws->stage[i], slot_bytes));
        }
        ws->stage_cap = slot_bytes;
    }
    if (ws->pin_cap < slot_bytes) {
        for (int i = 0; i < kSlots; ++i) {
            cudaFreeHost(ws->pin[i]);
            ws->pin[i] = nullptr;
            MPIC_CUDA(cudaMallocHost(&ws->pin[i], slot_bytes));
            if (!ws->ev_pin[i]) MPIC_CUDA(cudaEventCreateWithFlags(&ws->ev_pin[i], cudaEventDisableTiming));
        }
        ws->pin_cap = slot_bytes;
    }
    std::vector<uint32_t> ts(n_img);
    for (uint32_t i = 0; i < n_img; ++i) ts[i] = r.refs[i].rows;
    const AsmChunk* dc[2];
    const float2* dt[2];
    void* bufs[2] = {nullptr, nullptr};
    uint32_t n_tab = 0;
    for (int sl = 0; sl < 2; ++sl) {
        std::vector<const void*> ks(n_img), vs(n_img);
        char* base = static_cast<char*>(ws->stage[sl]);
        for (uint32_t i = 0; i < n_img; ++i) {
            ks[i] = base + off[i] * es;
            vs[i] = base + (img_rows * h + off[i]) * es;
        }
        const AsmPlan p = plan_assembly(ks.data(), vs.data(), ts.data(), r.refs.data(), n_img, linked->T, linked->D,
                                        reposition, model->cfg.rope_base, linked->H * linked->D);
        n_tab = p.n_tables;
        bufs[sl] = upload_plan(p, s, &dc[sl], &dt[sl]);
    }
    // compute lane: every chunk not loaded from its file, started before the first load
    MissLane lane(model, ws);
    for (uint32_t i = 0; i < n_img; ++i)
        if (status[i] != MPIC_CHUNK_LOADED) lane.start(i, hashes[i], r.refs[i].rows);

    // reader threads: layer l -> pinned slot l % kSlots, per-piece CRCs; the thread that
    // completes a layer checks the v3 per-layer CRCs of every chunk before the layer is
    // handed to the copy stream
    std::vector<uint32_t> loaded;
    for (uint32_t i = 0; i < n_img; ++i)
        if (status[i] == MPIC_CHUNK_LOADED) loaded.push_back(i);
    std::mutex mu;
    std::condition_variable cv;
    int filled = -1;  // highest layer whose pinned slot is complete and verified
    std::vector<bool> copied(L, false);
    std::vector<uint32_t> done(L, 0);
    std::string reader_error;
    int bad_chunk = -1;  // a loaded chunk that failed verification (or its read)
    const uint32_t n_seg = 2 * (uint32_t)loaded.size();
    const uint32_t hw = std::max<uint32_t>(1, std::thread::hardware_concurrency());
    const uint32_t want = std::max<uint32_t>(1, hw > 4 ? hw - 2 : hw);
    const uint32_t pieces = n_seg ? std::max<uint32_t>(1, std::min<uint32_t>(8, ceil_div(want, n_seg))) : 1;
    const uint32_t n_items = n_seg * pieces;
    const uint32_t n_threads = n_items ? std::max<uint32_t>(1, std::min<uint32_t>(n_items, want)) : 0;
    for (uint32_t i : loaded) files[i]->crc_piece.assign(2 * (size_t)L * pieces, 0);
    // CRCs on the GPU (default): every loaded layer is checksummed in HBM right after its H2D,
    // on the copy stream, so the reader threads only move bytes (the host CRC pass cost ~45% of
    // a page-cache-warm request at config C); the per-layer (v3) and file CRCs are compared
    // once the request has run, and a mismatch re-runs it with that chunk computed — as for a
    // v1/v2 file CRC — so the outputs never come from corrupt bytes. MPIC_FILES_CRC=host checks
    // on the reader threads before each H2D instead.
    static const bool gpu_crc_env = [] {
        const char* e = getenv("MPIC_FILES_CRC");
        return !(e && std::string(e) == "host");
    }();
    const bool gpu_crc = gpu_crc_env;
    constexpr uint32_t kFilePiece = 128 * 1024;
    std::vector<size_t> pc_off(n_img, 0);  // chunk i's first piece in d_pcrc ([2][L][ppp_i])
    size_t n_pc = 0;
    for (uint32_t i : loaded) {
        pc_off[i] = n_pc;
        n_pc += 2 * (size_t)L * ceil_div((size_t)files[i]->T * h * es, (size_t)kFilePiece);
    }
    uint32_t* d_pcrc = nullptr;
    if (gpu_crc && n_pc) MPIC_CUDA(cudaMallocAsync((void**)&d_pcrc, n_pc * 4, ws->copy_stream));
    auto seg_crc = [&](const MpicFile& f, uint32_t is_v, uint32_t l) {
        const size_t seg = (size_t)f.T * h * es;
        if (gpu_crc) return f.layer_crc[is_v * L + l];
        uLong c = f.crc_piece[((size_t)is_v * L + l) * pieces];
        for (uint32_t pc = 1; pc < pieces; ++pc) {
            const size_t p0 = seg * pc / pieces, p1 = seg * (pc + 1) / pieces;
            c = crc32_combine(c, f.crc_piece[((size_t)is_v * L + l) * pieces + pc], (z_off_t)(p1 - p0));
        }
        return (uint32_t)c;
    };
    auto read_worker = [&](uint32_t w) {
        uint32_t cur = 0;
        try {
            for (uint32_t l = 0; l < L; ++l) {
                const int sl = (int)(l % kSlots);
                if (l >= (uint32_t)kSlots) {  // wait for the H2D that last used this slot
                    std::unique_lock<std::mutex> lk(mu);
                    cv.wait(lk, [&] { return copied[l - kSlots] || !reader_error.empty(); });
                    if (!reader_error.empty()) return;
                    lk.unlock();
                    MPIC_CUDA(cudaEventSynchronize(ws->ev_pin[sl]));
                }
                char* dst = static_cast<char*>(ws->pin[sl]);
                for (uint32_t it = w; it < n_items; it += n_threads) {
                    const uint32_t sg = it / pieces, pc = it % pieces;
                    const uint32_t i = loaded[sg >> 1];
                    cur = i;
                    const uint32_t is_v = sg & 1;
                    MpicFile& f = *files[i];
                    const size_t seg = (size_t)f.T * h * es;
                    const size_t p0 = seg * pc / pieces, p1 = seg * (pc + 1) / pieces;
                    char* d = dst + ((is_v ? img_rows * h : 0) + off[i]) * es + p0;
                    pread_all(f.fd, d, p1 - p0, (off_t)(84 + ((is_v ? (size_t)L : 0) + l) * seg + p0));
                    if (!gpu_crc) f.crc_piece[((size_t)is_v * L + l) * pieces + pc] = crc_of(d, p1 - p0);
                }
                {
                    std::lock_guard<std::mutex> lk(mu);
                    if (++done[l] == n_threads) {
                        for (uint32_t i : loaded) {  // v3: verify the layer before it is used
                            const MpicFile& f = *files[i];
                            if (f.version == 3 && bad_chunk < 0 && !gpu_crc &&
                                (seg_crc(f, 0, l) != f.table[l] || seg_crc(f, 1, l) != f.table[L + l]))
                                bad_chunk = (int)i;
                        }
                        filled = (int)l;
                    }
                }
                cv.notify_all();
            }
        } catch (const Error&) {  // a short read: the chunk falls back to the compute lane
            std::lock_guard<std::mutex> lk(mu);
            if (bad_chunk < 0) bad_chunk = (int)cur;
            reader_error = "read failure";
            cv.notify_all();
        } catch (const std::exception& e) {
            std::lock_guard<std::mutex> lk(mu);
            reader_error = e.what();
            cv.notify_all();
        }
    };
    std::vector<std::thread> readers;
    for (uint32_t w = 0; w < n_threads; ++w) readers.emplace_back(read_worker, w);
    auto stop_readers = [&] {
        {
            std::lock_guard<std::mutex> lk(mu);
            if (reader_error.empty()) reader_error = "request aborted";
            for (uint32_t l = 0; l < L; ++l) copied[l] = true;
        }
        cv.notify_all();
        for (std::thread& t : readers) t.join();
        readers.clear();
    };
    const size_t e = esz(linked->dtype);
    const size_t plane = (size_t)linked->T * h * e;
    cudaStream_t cs = ws->copy_stream;
    MPIC_CUDA(cudaEventRecord(ws->ev_free[0], s));
    MPIC_CUDA(cudaEventRecord(ws->ev_free[1], s));
    auto issue_copy = [&](uint32_t l) {
        if (n_threads) {
            std::unique_lock<std::mutex> lk(mu);
            cv.wait(lk, [&] { return filled >= (int)l || bad_chunk >= 0 || !reader_error.empty(); });
            if (bad_chunk >= 0) throw RerunWithCompute{(uint32_t)bad_chunk};
            if (!reader_error.empty()) throw Error(MPIC_ERR_IO, "disk loader: " + reader_error);
        }
        const int sl = l & 1, ps = (int)(l % kSlots);
        char* stage = static_cast<char*>(ws->stage[sl]);
        MPIC_CUDA(cudaStreamWaitEvent(cs, ws->ev_free[sl], 0));
        if (loaded_rows) {
            const char* pin = static_cast<const char*>(ws->pin[ps]);
            const size_t lb = loaded_rows * h * es, vo = img_rows * h * es;
            MPIC_CUDA(cudaMemcpyAsync(stage, pin, lb, cudaMemcpyHostToDevice, cs));
            MPIC_CUDA(cudaMemcpyAsync(stage + vo, pin + vo, lb, cudaMemcpyHostToDevice, cs));
        }
        MPIC_CUDA(cudaEventRecord(ws->ev_pin[ps], cs));
        for (const auto& j : lane.jobs)
            lane.copy_layer(*j, l, stage + off[j->chunk] * es, stage + (img_rows * h + off[j->chunk]) * es, ct, cs);
        MPIC_CUDA(cudaEventRecord(ws->ev_ready[sl], cs));
        if (d_pcrc)  // this layer's loaded K / V planes, checksummed in HBM behind the copy
            for (uint32_t i : loaded) {
                const size_t seg = (size_t)files[i]->T * h * es, ppp = ceil_div(seg, (size_t)kFilePiece);
                launch_crc32_pieces(stage + off[i] * es, seg, 1, kFilePiece, d_pcrc + pc_off[i] + l * ppp, cs);
                launch_crc32_pieces(stage + (img_rows * h + off[i]) * es, seg, 1, kFilePiece,
                                    d_pcrc + pc_off[i] + (L + l) * ppp, cs);
            }
        if (n_threads) {
            std::lock_guard<std::mutex> lk(mu);
            copied[l] = true;
        }
        cv.notify_all();
    };
    auto before_layer = [&](uint32_t l) {
        if (l + 1 < L) issue_copy(l + 1);
        const int sl = l & 1;
        MPIC_CUDA(cudaStreamWaitEvent(s, ws->ev_ready[sl], 0));
        ProfScope ps(s, MPIC_PHASE_ASSEMBLE);
        launch_assemble(dc[sl], n_img, dt[sl], n_tab, ct, (char*)linked->k + l * plane, (char*)linked->v + l * plane,
                        linked->dtype, 1, linked->T, linked->H, linked->D, 1, s);
        MPIC_CUDA(cudaEventRecord(ws->ev_free[sl], s));
    };
    auto drain = [&] {  // nothing of this pass may still touch the rings when it returns
        cudaStreamSynchronize(s);
        cudaStreamSynchronize(cs);
        for (int sl = 0; sl < 2; ++sl) cudaFreeAsync(bufs[sl], s);
        if (d_pcrc) cudaFreeAsync(d_pcrc, cs);
    };
    try {
        issue_copy(0);
        run_request(model, ws, r, linked, logits, selected, m_out, s, before_layer);
    } catch (const RerunWithCompute& rr) {
        stop_readers();
        drain();
        return (int)rr.chunk;
    } catch (...) {
        stop_readers();
        drain();
        throw;
    }
    for (std::thread& t : readers) t.join();
    for (int sl = 0; sl < 2; ++sl) MPIC_CUDA(cudaFreeAsync(bufs[sl], s));
    if (d_pcrc) {
        std::vector<uint32_t> hp(n_pc);
        MPIC_CUDA(cudaMemcpyAsync(hp.data(), d_pcrc, n_pc * 4, cudaMemcpyDeviceToHost, cs));
        MPIC_CUDA(cudaFreeAsync(d_pcrc, cs));
        MPIC_CUDA(cudaStreamSynchronize(cs));
        for (uint32_t i : loaded) {
            MpicFile& f = *files[i];
            const size_t seg = (size_t)f.T * h * es, ppp = ceil_div(seg, (size_t)kFilePiece);
            f.layer_crc.resize(2 * L);
            for (uint32_t q = 0; q < 2 * L; ++q)
                f.layer_crc[q] = combine_crc_pieces(hp.data() + pc_off[i] + q * ppp, seg, kFilePiece);
            if (f.version == 3 && bad_chunk < 0)
                for (uint32_t q = 0; q < 2 * L; ++q)
                    if (f.layer_crc[q] != f.table[q]) {
                        bad_chunk = (int)i;
                        break;
                    }
        }
    }
    if (bad_chunk >= 0) return bad_chunk;
    MPIC_REQUIRE(reader_error.empty(), MPIC_ERR_IO, "disk loader: " + reader_error);
    for (uint32_t i : loaded) {  // CRC of the whole file, in file order (v1/v2: the only check)
        MpicFile& f = *files[i];
        const size_t seg = (size_t)f.T * h * es;
        uLong c = f.crc_header;
        for (uint32_t is_v = 0; is_v < 2; ++is_v)
            for (uint32_t l = 0; l < L; ++l) c = crc32_combine(c, seg_crc(f, is_v, l), (z_off_t)seg);
        if (f.version == 3) c = crc32(c, reinterpret_cast<const Bytef*>(f.table.data()), (uInt)(f.table.size() * 4));
        if ((uint32_t)c != f.crc_stored) return (int)i;
    }
    return -1;
}
}  // namespace

int mpic_request_prefill_files2(mpic_model_t model, mpic_workspace_t ws, const mpic_prompt* prompt,
                                const mpic_policy* policy, const char* const* paths, mpic_reposition reposition,
                                mpic_kv_t linked, float* logits, uint32_t* selected, uint32_t* m_out,
                                uint32_t* chunk_status, void* stream) {
    API_BEGIN
    MPIC_CUDA(cudaSetDevice(model->device));
    cudaStream_t s = (cudaStream_t)stream;
    const RequestPlan r0 = plan_request(model, prompt, policy, nullptr);
    check_linked(model, linked, r0.n);
    const uint32_t n_img = (uint32_t)r0.refs.size();
    const std::vector<const uint8_t*> hashes = image_hashes(prompt);
    std::vector<std::unique_ptr<MpicFile>> files(n_img);
    std::vector<uint32_t> status(n_img, MPIC_CHUNK_LOADED);
    for (uint32_t i = 0; i < n_img; ++i) {  // the store lookup (split_request, transfer.cpp:65-79)
        if (!paths || !paths[i]) {
            status[i] = MPIC_CHUNK_COMPUTED;
            continue;
        }
        files[i] = std::make_unique<MpicFile>();
        try {
            open_mpic(*files[i], paths[i], model, r0.refs[i].rows, hashes[i]);
        } catch (const Error& e) {
            status[i] = e.code == MPIC_ERR_NOT_FOUND ? MPIC_CHUNK_COMPUTED : MPIC_CHUNK_FALLBACK;
            files[i].reset();
        }
    }
    for (uint32_t attempt = 0;; ++attempt) {
        const int bad = files_pass(model, ws, prompt, policy, paths, reposition, linked, logits, selected, m_out, s,
                                   status, files);
        if (bad < 0) break;
        MPIC_REQUIRE(attempt < n_img, MPIC_ERR_STATE, "disk loader: re-run did not converge");
        status[bad] = MPIC_CHUNK_FALLBACK;
        files[bad].reset();
    }
    if (chunk_status) std::memcpy(chunk_status, status.data(), n_img * sizeof(uint32_t));
    API_END
}

int mpic_request_prefill_files(mpic_model_t model, mpic_workspace_t ws, const mpic_prompt* prompt,
                               const mpic_policy* policy, const char* const* paths, mpic_reposition reposition,
                               mpic_kv_t linked, float* logits, uint32_t* selected, uint32_t* m_out, void* stream) {
    return mpic_request_prefill_files2(model, ws, prompt, policy, paths, reposition, linked, logits, selected, m_out,
                                       nullptr, stream);
}

int mpic_test_gemm(const void* d_a, const void* d_w, uint32_t M, uint32_t N, uint32_t K,
                   int path, float* d_out, void* stream) {
    API_BEGIN
    EpiParams ep;
    ep.mode = EPI_STORE_F32;
    ep.out = d_out;
    ep.ldo = N;
    cudaStream_t s = (cudaStream_t)stream;
    if (path == 1) {
        MPIC_REQUIRE(tc_gemm_supported(M, N, K), MPIC_ERR_VALIDATION, "shape not supported by the tcgen05 gemm");
        launch_gemm_tc(static_cast<const __nv_bfloat16*>(d_a), K, static_cast<const __nv_bfloat16*>(d_w), M, N, K, ep, s);
    } else if (path == 3) {  // d_w already in the blocked layout
        launch_gemm_tc(static_cast<const __nv_bfloat16*>(d_a), K, static_cast<const __nv_bfloat16*>(d_w), M, N, K, ep, s,
                       true);
    } else if (path == 2) {  // the same weights in the blocked layout
        MPIC_REQUIRE(pgemm_supported(M, N, K), MPIC_ERR_VALIDATION, "shape not supported by the pair gemm");
        __nv_bfloat16* wb = nullptr;
        MPIC_CUDA(cudaMallocAsync((void**)&wb, (size_t)N * K * 2, s));
        launch_block_weights(static_cast<const __nv_bfloat16*>(d_w), wb, N, K, true, s);
        launch_gemm_tc(static_cast<const __nv_bfloat16*>(d_a), K, wb, M, N, K, ep, s, true);
        MPIC_CUDA(cudaFreeAsync(wb, s));
    } else if (path == 4 || path == 5) {  // fp32 operands: 4 = 3xTF32 pair gemm, 5 = SIMT FFMA
        if (path == 5) {
            launch_gemm_simt(d_a, MPIC_F32, K, d_w, MPIC_F32, M, N, K, ep, MPIC_F32, s);
        } else {
            MPIC_REQUIRE(pgemm_x3_supported(M, N, K), MPIC_ERR_VALIDATION, "shape not supported by the 3xTF32 gemm");
            float* buf = nullptr;
            const size_t na = (size_t)M * K, nw = (size_t)N * K;
            MPIC_CUDA(cudaMallocAsync((void**)&buf, (2 * na + 2 * nw) * 4, s));
            launch_tf32_split(static_cast<const float*>(d_a), buf, buf + na, na, s);
            launch_tf32_split(static_cast<const float*>(d_w), buf + 2 * na, buf + 2 * na + nw, nw, s);
            launch_pgemm_x3(buf, buf + na, buf + 2 * na, buf + 2 * na + nw, M, N, K, ep, s);
            MPIC_CUDA(cudaFreeAsync(buf, s));
        }
    } else {
        launch_gemm_simt(d_a, MPIC_BF16, K, d_w, MPIC_BF16, M, N, K, ep, MPIC_BF16, s);
    }
    API_END
}

int mpic_test_gemm_epi(const void* d_a, const void* d_w, uint32_t M, uint32_t N, uint32_t K, int mode,
                       float* d_x, void* d_xb, void* d_out, void* stream) {
    API_BEGIN
    MPIC_REQUIRE(tc_gemm_supported(M, N, K), MPIC_ERR_VALIDATION, "shape not supported by the tcgen05 gemm");
    EpiParams ep;
    if (mode == 3) {  // EPI_QKV with head_dim 128 (timing): q -> d_out, K/V scattered to rows 0..M-1 of
                      // scratch planes, zero (cos, sin) rows. The scratch is made on the first (uncaptured) call.
        const uint32_t h = N / 3;
        const size_t plane = (size_t)M * h * 2, rope = (size_t)M * 64 * sizeof(float2), rows = (size_t)M * 4;
        static char* b = nullptr;
        static size_t cap = 0;
        if (cap < 2 * plane + rope + rows) {
            cudaFree(b);
            MPIC_CUDA(cudaMalloc(&b, 2 * plane + rope + rows));
            cap = 2 * plane + rope + rows;
            MPIC_CUDA(cudaMemset(b + 2 * plane, 0, rope));
            std::vector<uint32_t> ident(M);
            for (uint32_t i = 0; i < M; ++i) ident[i] = i;
            MPIC_CUDA(cudaMemcpy(b + 2 * plane + rope, ident.data(), rows, cudaMemcpyHostToDevice));
        }
        ep.mode = EPI_QKV;
        ep.q = d_out;
        ep.kv_k = b;
        ep.kv_v = b + plane;
        ep.rope_tok = reinterpret_cast<const float2*>(b + 2 * plane);
        ep.kv_rows = reinterpret_cast<const uint32_t*>(b + 2 * plane + rope);
        ep.rope_pos = ep.kv_rows;
        ep.hidden = h;
        ep.head_dim = 128;
    } else if (mode == 0) {
        ep.mode = EPI_RESID;
        ep.x = d_x;
        ep.xb = static_cast<__nv_bfloat16*>(d_xb);
        ep.ldx = N;
    } else {
        ep.mode = mode == 1 ? EPI_GELU : EPI_STORE;
        ep.out = d_out;
        ep.ldo = N;
    }
    launch_gemm_tc(static_cast<const __nv_bfloat16*>(d_a), K, static_cast<const __nv_bfloat16*>(d_w), M, N, K, ep,
                   (cudaStream_t)stream);
    API_END
}

int mpic_test_qkv(const void* d_a, const void* d_w, uint32_t M, uint32_t h, uint32_t K, uint32_t head_dim,
                  const uint32_t* d_rows, const void* d_rope_tok, void* d_q, void* d_kv_k, void* d_kv_v,
                  void* stream) {
    API_BEGIN
    MPIC_REQUIRE(tc_gemm_supported(M, 3 * h, K), MPIC_ERR_VALIDATION, "shape not supported by the tcgen05 gemm");
    EpiParams ep;
    ep.mode = EPI_QKV;
    ep.q = d_q;
    ep.kv_k = d_kv_k;
    ep.kv_v = d_kv_v;
    ep.kv_rows = d_rows;
    ep.rope_pos = d_rows;
    ep.rope_tok = static_cast<const float2*>(d_rope_tok);
    ep.hidden = h;
    ep.head_dim = head_dim;
    launch_gemm_tc(static_cast<const __nv_bfloat16*>(d_a), K, static_cast<const __nv_bfloat16*>(d_w), M, 3 * h, K,
                   ep, (cudaStream_t)stream);
    API_END
}

int mpic_pgemm_timestamps(unsigned long long* out9) {
    API_BEGIN
    pgemm_timestamps(out9);
    API_END
}

int mpic_clock_probe(float* d_out_mhz, uint32_t spin_ns, void* stream) {
    API_BEGIN
    launch_clock_probe(d_out_mhz, spin_ns, (cudaStream_t)stream);
    API_END
}

int mpic_profile_enable(int on) {
    API_BEGIN
    std::lock_guard<std::mutex> lk(g_prof_mu);
    g_prof_on = on != 0;
    API_END
}

int mpic_profile_collect(double* ms, uint32_t* launches) {
    API_BEGIN
    std::vector<ProfRec> recs;
    {
        std::lock_guard<std::mutex> lk(g_prof_mu);
        recs.swap(g_prof_recs);
    }
    for (int i = 0; i < MPIC_PHASE_COUNT; ++i) {
        ms[i] = 0.0;
        launches[i] = 0;
    }
    for (const ProfRec& r : recs) {
        MPIC_CUDA(cudaEventSynchronize(r.b));
        float t = 0.f;
        MPIC_CUDA(cudaEventElapsedTime(&t, r.a, r.b));
        ms[r.cls] += t;
        launches[r.cls] += 1;
    }
    std::lock_guard<std::mutex> lk(g_prof_mu);
    for (const ProfRec& r : recs) {
        g_prof_pool.push_back(r.a);
        g_prof_pool.push_back(r.b);
    }
    API_END
}

int mpic_attention_plan(const uint32_t* rows, uint32_t m, uint32_t n_heads, const uint32_t* starts,
                        uint32_t* counts, uint32_t* units_out, uint32_t units_cap, uint32_t* offs_out,
                        uint32_t offs_cap, uint32_t* jobs_out, uint32_t jobs_cap) {
    API_BEGIN
    MPIC_REQUIRE(rows && counts && m > 0 && n_heads > 0, MPIC_ERR_VALIDATION, "attention plan: bad arguments");
    const AttnPlan plan = plan_attention(rows, m, n_heads, starts);
    const uint32_t ctas = std::min<uint32_t>(plan.items, kNumSMs);
    counts[0] = plan.items;
    counts[1] = ctas;
    counts[2] = (uint32_t)plan.combine.size();
    counts[3] = plan.slots;
    static_assert(sizeof(AttnUnit) == 10 * sizeof(uint32_t), "AttnUnit layout");
    if (units_out) {
        MPIC_REQUIRE(units_cap >= plan.items, MPIC_ERR_VALIDATION, "attention plan: units_out too small");
        std::memcpy(units_out, plan.units.data(), (size_t)plan.items * sizeof(AttnUnit));
    }
    if (offs_out) {
        MPIC_REQUIRE(offs_cap >= ctas + 1, MPIC_ERR_VALIDATION, "attention plan: offs_out too small");
        std::memcpy(offs_out, attn_cta_offsets(plan.units.data(), plan.items), (ctas + 1) * sizeof(uint32_t));
    }
    if (jobs_out) {
        MPIC_REQUIRE(jobs_cap >= plan.combine.size(), MPIC_ERR_VALIDATION, "attention plan: jobs_out too small");
        std::memcpy(jobs_out, plan.combine.data(), plan.combine.size() * sizeof(AttnCombine));
    }
    API_END
}

int mpic_test_attention(const void* d_q, const void* d_k, const void* d_v, const uint32_t* rows,
                        uint32_t m, uint32_t n_ctx, uint32_t n_heads, void* d_out, void* stream) {
    API_BEGIN
    cudaStream_t s = (cudaStream_t)stream;
    const AttnPlan plan = plan_attention(rows, m, n_heads);
    void* buf = nullptr;
    auto al = [](size_t x) { return (x + 255) / 256 * 256; };
    const size_t bu = al(plan.units.size() * sizeof(AttnUnit)), bc = al(plan.combine.size() * sizeof(AttnCombine));
    const size_t bo = al((size_t)plan.slots * 128 * 128 * 4), bm = al((size_t)plan.slots * 128 * 8), br = al((size_t)m * 4);
    const size_t bn = (size_t)plan.combine.size() * 4;
    MPIC_CUDA(cudaMallocAsync(&buf, bu + bc + bo + bm + br + bn + 64, s));
    char* b = static_cast<char*>(buf);
    uint32_t* d_cnt = !fused_combine() || !bn ? nullptr : reinterpret_cast<uint32_t*>(b + bu + bc + bo + bm + br);
    if (d_cnt) MPIC_CUDA(cudaMemsetAsync(d_cnt, 0, bn, s));
    MPIC_CUDA(cudaMemcpyAsync(b, plan.units.data(), plan.units.size() * sizeof(AttnUnit), cudaMemcpyHostToDevice, s));
    if (!plan.combine.empty())
        MPIC_CUDA(cudaMemcpyAsync(b + bu, plan.combine.data(), plan.combine.size() * sizeof(AttnCombine),
                                  cudaMemcpyHostToDevice, s));
    MPIC_CUDA(cudaMemcpyAsync(b + bu + bc + bo + bm, rows, br, cudaMemcpyHostToDevice, s));
    launch_attn_tc(static_cast<const __nv_bfloat16*>(d_q), static_cast<const __nv_bfloat16*>(d_k),
                   static_cast<const __nv_bfloat16*>(d_v), n_ctx,
                   reinterpret_cast<const uint32_t*>(b + bu + bc + bo + bm), m, n_heads,
                   reinterpret_cast<const AttnUnit*>(b), plan.items,
                   reinterpret_cast<const AttnCombine*>(b + bu), (uint32_t)plan.combine.size(),
                   reinterpret_cast<float*>(b + bu + bc), reinterpret_cast<float2*>(b + bu + bc + bo),
                   static_cast<__nv_bfloat16*>(d_out), s, nullptr, 0, nullptr, d_cnt);
    MPIC_CUDA(cudaFreeAsync(buf, s));
    if (unsigned long long* dbg = attn_debug_buffer()) {  // MPIC_ATTN_TS diagnostics
        std::vector<unsigned long long> h(16 * 4096);
        MPIC_CUDA(cudaStreamSynchronize(s));
        MPIC_CUDA(cudaMemcpy(h.data(), dbg, h.size() * 8, cudaMemcpyDeviceToHost));
        MPIC_CUDA(cudaMemset(dbg, 0, h.size() * 8));
        {  // per-CTA spans (start, end, smid, first MMA, last burst, epilogue start/end), relative to the earliest start
            const size_t base = 16 * 64, ncta = std::min<size_t>(std::min<size_t>(plan.items, kNumSMs), (h.size() - base) / 8);
            const uint32_t* offs = attn_cta_offsets(plan.units.data(), plan.items);
            unsigned long long t_min = ~0ull;
            for (size_t c = 0; c < ncta; ++c) t_min = std::min(t_min, h[base + 8 * c]);
            auto rel = [&](size_t c, int k) { return h[base + 8 * c + k] ? (h[base + 8 * c + k] - t_min) / 1e3 : -1.0; };
            for (size_t c = 0; c < ncta; ++c) {
                const AttnUnit& u = plan.units[offs[c]];  // the CTA's first item
                fprintf(stderr, "cta %4zu sm %3llu start %8.2f end %8.2f us  head %u b0 %u tiles %u/%u b1 %u/%u | mma0 %8.2f "
                                "lastmma %8.2f epi %8.2f epi_end %8.2f\n", c,
                        h[base + 8 * c + 2], rel(c, 0), rel(c, 1), u.head, u.b0, u.tile[0], u.tile[1] == kNoTile ? 999u : u.tile[1],
                        u.b1[0], u.b1[1], rel(c, 3), rel(c, 4), rel(c, 5), rel(c, 6));
            }
        }
        const AttnUnit& u0 = plan.units[0];
        fprintf(stderr, "attn CTA0 item: head %u b0 %u tiles %u/%u b1 %u/%u\n", u0.head, u0.b0, u0.tile[0], u0.tile[1],
                u0.b1[0], u0.b1[1]);
        const long long t0 = (long long)h[0];
        auto at = [&](int j, int k) { return h[j * 16 + k] ? ((long long)h[j * 16 + k] - t0) / 1e3 : -1.0; };
        for (int j = 1; j < 64 && h[j * 16]; ++j)
            if (h[j * 16 + 14] && h[(j - 1) * 16 + 14])
                fprintf(stderr, "step %d: SM clock %.0f MHz\n", j,
                        1e3 * (double)(h[j * 16 + 14] - h[(j - 1) * 16 + 14]) / (double)(h[j * 16] - h[(j - 1) * 16]));
        for (int j = 0; j < 64 && h[j * 16]; ++j)
            fprintf(stderr, "j=%2d MMA: start %6.2f pA %6.2f vA %6.2f pB %6.2f vB %6.2f deps %6.2f issued %6.2f | softmax A: S %6.2f "
                            "loaded %6.2f max %6.2f exps %6.2f P %6.2f | softmax B: S %6.2f P %6.2f us\n",
                    j, at(j, 0), at(j, 3), at(j, 12), at(j, 4), at(j, 13), at(j, 1), at(j, 2), at(j, 5), at(j, 8), at(j, 7),
                    at(j, 9), at(j, 6), at(j, 10), at(j, 11));
    }
    API_END
}

int mpic_host_gemm_f32(const float* a, const float* b, uint32_t M, uint32_t N, uint32_t K, float* c,
                       int device) {
    API_BEGIN
    set_device(device);
    float *da = nullptr, *db = nullptr, *dc = nullptr;
    cudaStream_t s = 0;
    MPIC_CUDA(cudaMalloc(&da, std::max<size_t>(1, (size_t)M * K) * 4));
    MPIC_CUDA(cudaMalloc(&db, std::max<size_t>(1, (size_t)N * K) * 4));
    MPIC_CUDA(cudaMalloc(&dc, std::max<size_t>(1, (size_t)M * N) * 4));
    MPIC_CUDA(cudaMemcpy(da, a, (size_t)M * K * 4, cudaMemcpyHostToDevice));
    MPIC_CUDA(cudaMemcpy(db, b, (size_t)N * K * 4, cudaMemcpyHostToDevice));
    EpiParams ep;
    ep.mode = EPI_STORE_F32;
    ep.out = dc;
    ep.ldo = N;
    launch_gemm_simt(da, MPIC_F32, K, db, MPIC_F32, M, N, K, ep, MPIC_F32, s);
    MPIC_CUDA(cudaMemcpy(c, dc, (size_t)M * N * 4, cudaMemcpyDeviceToHost));
    cudaFree(da);
    cudaFree(db);
    cudaFree(dc);
    API_END
}

int mpic_host_alloc(size_t bytes, void** out) {
    API_BEGIN
    MPIC_CUDA(cudaMallocHost(out, bytes));
    API_END
}

int mpic_host_free(void* p) {
    API_BEGIN
    MPIC_CUDA(cudaFreeHost(p));
    API_END
}

}  // extern "C"
