// Tiered chunk store on the device: the reference's CacheStore
// (proj/include/mpic/cache.h:70-133, proj/src/cache.cpp:203-461) with the Device tier in HBM
// (mpic_kv_t tensors in the model dtype), the Host tier in pinned memory and the Disk tier
// as .mpic v3 files (per-layer CRCs), LRU demotion by entry-count budgets
// (enforce_budgets_locked / demote_one_locked, cache.cpp:426-461), and a request entry that
// fetches (promotes to Device) every image chunk of a prompt and runs the device-resident
// MPIC request on them (prepare + selective_prefill, transfer.cpp:83-145).
//
// Integrity on the device: the per-layer CRC32 of every entry is computed by a GPU kernel
// over the stored bytes when the entry enters the store; a Host- or Disk-tier entry is
// re-checked on the device after its H2D, before the request uses it, and a mismatch (or an
// unreadable / foreign file) makes the chunk a fallback: it is computed (compute_entry,
// transfer.cpp:41-58) as a miss is. Demotion to Disk writes the file from the stored CRCs
// (zlib crc32_combine): no host pass over the payload.
//
// Built over the public C ABI (mpic_b200.h) plus the CRC kernel; host logic only otherwise.
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>
#include <zlib.h>

#include <array>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"
#include "kernels.h"

struct mpic_store_s;

namespace mpicb {
namespace {

// ---- CRC32 (zlib polynomial) of device memory: one thread per piece, slice-by-8 ----------
__global__ void crc32_pieces_kernel(const uint8_t* __restrict__ base, size_t plane_bytes, uint32_t n_planes,
                                    uint32_t piece, uint32_t* __restrict__ out) {
    __shared__ uint32_t tab[8][256];
    for (uint32_t i = threadIdx.x; i < 256; i += blockDim.x) {
        uint32_t c = i;
        for (int k = 0; k < 8; ++k) c = (c >> 1) ^ (0xEDB88320u & (0u - (c & 1u)));
        tab[0][i] = c;
    }
    __syncthreads();
    for (uint32_t s = 1; s < 8; ++s) {
        for (uint32_t i = threadIdx.x; i < 256; i += blockDim.x)
            tab[s][i] = (tab[s - 1][i] >> 8) ^ tab[0][tab[s - 1][i] & 0xFFu];
        __syncthreads();
    }
    const uint64_t ppp = (plane_bytes + piece - 1) / piece;
    const uint64_t idx = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (idx >= ppp * n_planes) return;
    const uint64_t plane = idx / ppp, j = idx % ppp;
    const size_t off = j * (size_t)piece;
    const size_t len = min((size_t)piece, plane_bytes - off);
    const uint8_t* p = base + plane * plane_bytes + off;
    uint32_t c = 0xFFFFFFFFu;
    size_t i = 0;
    if ((reinterpret_cast<uintptr_t>(p) & 7u) == 0) {
        for (; i + 8 <= len; i += 8) {
            const uint2 w = *reinterpret_cast<const uint2*>(p + i);
            const uint32_t a = w.x ^ c, b = w.y;
            c = tab[7][a & 0xFFu] ^ tab[6][(a >> 8) & 0xFFu] ^ tab[5][(a >> 16) & 0xFFu] ^ tab[4][a >> 24] ^
                tab[3][b & 0xFFu] ^ tab[2][(b >> 8) & 0xFFu] ^ tab[1][(b >> 16) & 0xFFu] ^ tab[0][b >> 24];
        }
    }
    for (; i < len; ++i) c = (c >> 8) ^ tab[0][(c ^ p[i]) & 0xFFu];
    out[idx] = ~c;
}

constexpr uint32_t kCrcPiece = 32768;

// zlib-compatible CRC32 of each of n_planes consecutive planes of plane_bytes bytes at the
// device address base: the pieces on the GPU, their combination on the host.
std::vector<uint32_t> device_plane_crcs(const void* base, size_t plane_bytes, uint32_t n_planes, cudaStream_t s) {
    std::vector<uint32_t> out(n_planes, 0);
    if (!n_planes) return out;
    if (!plane_bytes) {
        for (auto& c : out) c = (uint32_t)crc32(0L, Z_NULL, 0);
        return out;
    }
    const uint64_t ppp = (plane_bytes + kCrcPiece - 1) / kCrcPiece;
    const uint64_t n = ppp * n_planes;
    uint32_t* d = nullptr;
    MPIC_CUDA(cudaMallocAsync((void**)&d, n * 4, s));
    crc32_pieces_kernel<<<(uint32_t)((n + 255) / 256), 256, 0, s>>>(static_cast<const uint8_t*>(base), plane_bytes,
                                                                       n_planes, kCrcPiece, d);
    MPIC_LAUNCHED();
    std::vector<uint32_t> h(n);
    MPIC_CUDA(cudaMemcpyAsync(h.data(), d, n * 4, cudaMemcpyDeviceToHost, s));
    MPIC_CUDA(cudaFreeAsync(d, s));
    MPIC_CUDA(cudaStreamSynchronize(s));
    const uLong op = crc32_combine_gen((z_off_t)kCrcPiece);
    const size_t tail = plane_bytes - (ppp - 1) * (size_t)kCrcPiece;
    for (uint32_t pl = 0; pl < n_planes; ++pl) {
        uLong c = h[pl * ppp];
        for (uint64_t j = 1; j < ppp; ++j)
            c = j + 1 < ppp ? crc32_combine_op(c, h[pl * ppp + j], op)
                            : crc32_combine(c, h[pl * ppp + j], (z_off_t)tail);
        out[pl] = (uint32_t)c;
    }
    return out;
}

}  // namespace

// Warp per piece of 32 x 4 KB (the last piece of a plane may hold fewer): lane i checksums
// sub-piece i with four 16-B loads in flight, lane 0 folds the 32 sub-CRCs with the
// "append 4 KB" operator (zlib crc32_combine as a GF(2) matrix, m4k[j] = image of bit j).
// plane_bytes % 4096 == 0.
__constant__ uint32_t c_m4k[32];
__global__ void __launch_bounds__(128) crc32_warp_kernel(const uint8_t* __restrict__ base, size_t plane_bytes,
                                                         uint32_t n_planes, uint32_t* __restrict__ out) {
    __shared__ uint32_t tab[8][256];
    for (uint32_t i = threadIdx.x; i < 256; i += blockDim.x) {
        uint32_t c = i;
        for (int k = 0; k < 8; ++k) c = (c >> 1) ^ (0xEDB88320u & (0u - (c & 1u)));
        tab[0][i] = c;
    }
    __syncthreads();
    for (uint32_t t = 1; t < 8; ++t) {
        for (uint32_t i = threadIdx.x; i < 256; i += blockDim.x)
            tab[t][i] = (tab[t - 1][i] >> 8) ^ tab[0][tab[t - 1][i] & 0xFFu];
        __syncthreads();
    }
    constexpr uint32_t kSub = 4096, kPiece = 32 * kSub;
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t ppp = (plane_bytes + kPiece - 1) / kPiece;
    const uint64_t w = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    if (w >= ppp * n_planes) return;
    const uint64_t plane = w / ppp, j = w % ppp;
    const size_t off = j * (size_t)kPiece;
    const uint32_t nsub = (uint32_t)(min((size_t)kPiece, plane_bytes - off) / kSub);
    uint32_t c = 0xFFFFFFFFu;
    if (lane < nsub) {
        const uint4* p = reinterpret_cast<const uint4*>(base + plane * plane_bytes + off + (size_t)lane * kSub);
        auto step8 = [&](uint32_t a, uint32_t b) {
            a ^= c;
            c = tab[7][a & 0xFFu] ^ tab[6][(a >> 8) & 0xFFu] ^ tab[5][(a >> 16) & 0xFFu] ^ tab[4][a >> 24] ^
                tab[3][b & 0xFFu] ^ tab[2][(b >> 8) & 0xFFu] ^ tab[1][(b >> 16) & 0xFFu] ^ tab[0][b >> 24];
        };
        for (uint32_t q = 0; q < kSub / 16; q += 4) {
            uint4 v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) v[u] = __ldg(p + q + u);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                step8(v[u].x, v[u].y);
                step8(v[u].z, v[u].w);
            }
        }
    }
    c = ~c;
    uint32_t acc = __shfl_sync(0xffffffffu, c, 0);
    for (uint32_t i = 1; i < nsub; ++i) {  // lane 0 (all lanes compute it: warp-uniform)
        uint32_t sh = 0;
#pragma unroll
        for (uint32_t b = 0; b < 32; ++b)
            if (acc >> b & 1u) sh ^= c_m4k[b];
        acc = sh ^ __shfl_sync(0xffffffffu, c, i);
    }
    if (lane == 0) out[w] = acc;
}

void launch_crc32_pieces(const void* base, size_t plane_bytes, uint32_t n_planes, uint32_t piece, uint32_t* d_out,
                         cudaStream_t s) {
    const uint64_t n = (plane_bytes + piece - 1) / piece * n_planes;
    if (!n) return;
    if (piece == 32 * 4096 && plane_bytes % 4096 == 0) {
        static std::mutex mu;
        static bool init[64] = {};
        int dev = 0;
        MPIC_CUDA(cudaGetDevice(&dev));
        std::lock_guard<std::mutex> lk(mu);
        if (!init[dev & 63]) {  // __constant__ memory is per device
            uint32_t m[32];
            const uLong op = crc32_combine_gen((z_off_t)4096);
            for (int b = 0; b < 32; ++b) m[b] = (uint32_t)crc32_combine_op(1uL << b, 0, op);
            MPIC_CUDA(cudaMemcpyToSymbol(c_m4k, m, sizeof(m)));
            init[dev & 63] = true;
        }
        crc32_warp_kernel<<<(uint32_t)((n * 32 + 127) / 128), 128, 0, s>>>(static_cast<const uint8_t*>(base),
                                                                            plane_bytes, n_planes, d_out);
    } else {
        crc32_pieces_kernel<<<(uint32_t)((n + 127) / 128), 128, 0, s>>>(static_cast<const uint8_t*>(base),
                                                                           plane_bytes, n_planes, piece, d_out);
    }
    MPIC_LAUNCHED();
}

uint32_t combine_crc_pieces(const uint32_t* h, size_t plane_bytes, uint32_t piece) {
    const uint64_t ppp = (plane_bytes + piece - 1) / piece;
    if (!ppp) return (uint32_t)crc32(0L, Z_NULL, 0);
    static thread_local std::pair<uint32_t, uLong> op{0, 0};
    if (op.first != piece) op = {piece, crc32_combine_gen((z_off_t)piece)};
    uLong c = h[0];
    const size_t tail = plane_bytes - (ppp - 1) * (size_t)piece;
    for (uint64_t j = 1; j < ppp; ++j)
        c = j + 1 < ppp ? crc32_combine_op(c, h[j], op.second) : crc32_combine(c, h[j], (z_off_t)tail);
    return (uint32_t)c;
}

namespace {

uint64_t fnv1a_bytes(const void* p, size_t n) {
    uint64_t h = 0xcbf29ce484222325ull;
    const uint8_t* b = static_cast<const uint8_t*>(p);
    for (size_t i = 0; i < n; ++i) {
        h ^= b[i];
        h *= 0x100000001b3ull;
    }
    return h;
}

std::string hex_of(const uint8_t* p, size_t n) {
    static const char* d = "0123456789abcdef";
    std::string s;
    for (size_t i = 0; i < n; ++i) {
        s += d[p[i] >> 4];
        s += d[p[i] & 15];
    }
    return s;
}

void check_rc(int rc) {
    if (rc != MPIC_OK) throw Error(rc, mpic_last_error());
}

}  // namespace
}  // namespace mpicb

using namespace mpicb;

struct StoreKey {
    std::array<uint8_t, 32> hash{};
    std::string ns;
    bool operator<(const StoreKey& o) const { return hash != o.hash ? hash < o.hash : ns < o.ns; }
};

struct StoreEntry {
    int tier = MPIC_TIER_DEVICE;
    mpic_kv_t kv = nullptr;      // Device tier
    void* hk = nullptr;          // Host tier: pinned K, V planes [L][T][h] in the model dtype
    void* hv = nullptr;
    std::vector<uint32_t> crc;   // crc_k[L], crc_v[L] of the model-dtype layer planes
    uint32_t T = 0, position_base = 0;
    uint64_t last_use = 0;
};

struct mpic_store_s {
    mpic_model_t model = nullptr;
    mpic_model_config cfg{};
    mpic_dtype dtype = MPIC_F32;
    int device = 0;
    std::string dir;
    uint32_t device_budget = 0, host_budget = 0;
    std::map<StoreKey, StoreEntry> index;
    uint64_t counter = 0;
    std::mutex mu;
    cudaStream_t s = nullptr;
    mpic_workspace_t aux = nullptr;  // compute lane for misses / fallbacks
    uint32_t aux_rows = 0;

    size_t plane_bytes(uint32_t T) const { return (size_t)T * cfg.hidden_dim * elt_size(dtype); }
    std::string path_for(const StoreKey& k) const {  // cache.cpp:198-201
        char fp[17];
        snprintf(fp, sizeof(fp), "%016llx", (unsigned long long)mpic_config_fingerprint(&cfg));
        return dir + "/" + hex_of(reinterpret_cast<const uint8_t*>(k.ns.data()), k.ns.size()) + "/" + fp + "/" +
               hex_of(k.hash.data(), 32) + ".mpic";
    }
    void free_entry(StoreEntry& e) {
        if (e.kv) mpic_kv_free(e.kv);
        if (e.hk) cudaFreeHost(e.hk);
        if (e.hv) cudaFreeHost(e.hv);
        e.kv = nullptr;
        e.hk = e.hv = nullptr;
    }
    // Per-layer CRCs of a device KV in the model dtype (the GPU kernel).
    std::vector<uint32_t> kv_crcs(mpic_kv_t kv, uint32_t T) {
        void *k, *v;
        check_rc(mpic_kv_device_ptrs(kv, &k, &v));
        std::vector<uint32_t> c = device_plane_crcs(k, plane_bytes(T), cfg.n_layers, s);
        const std::vector<uint32_t> cv = device_plane_crcs(v, plane_bytes(T), cfg.n_layers, s);
        c.insert(c.end(), cv.begin(), cv.end());
        return c;
    }

    void write_file(const StoreKey& key, const StoreEntry& e) {  // .mpic v3, cache.cpp:97-125
        const std::string path = path_for(key);
        for (size_t p = dir.size() + 1; p < path.size(); ++p)
            if (path[p] == '/') mkdir(path.substr(0, p).c_str(), 0755);
        const uint32_t L = cfg.n_layers;
        uint8_t h[84] = {};
        std::memcpy(h, "MPIC", 4);
        const uint32_t version = 3;
        const uint64_t fp = mpic_config_fingerprint(&cfg), nsh = fnv1a_bytes(key.ns.data(), key.ns.size());
        std::memcpy(h + 4, &version, 4);
        std::memcpy(h + 8, &fp, 8);
        std::memcpy(h + 16, &nsh, 8);
        std::memcpy(h + 24, key.hash.data(), 32);
        const uint32_t dims[5] = {e.position_base, L, e.T, cfg.n_heads, cfg.head_dim};
        std::memcpy(h + 56, dims, 20);
        h[76] = dtype == MPIC_BF16 ? 1 : 0;
        const size_t pb = plane_bytes(e.T);
        FILE* f = fopen((path + ".tmp").c_str(), "wb");
        MPIC_REQUIRE(f, MPIC_ERR_IO, "cannot write " + path);
        bool ok = fwrite(h, 1, 84, f) == 84;
        uLong crc = crc32(0L, h, 84);
        for (int part = 0; part < 2 && ok; ++part)
            for (uint32_t l = 0; l < L && ok; ++l) {
                ok = fwrite(static_cast<const char*>(part ? e.hv : e.hk) + l * pb, 1, pb, f) == pb;
                crc = crc32_combine(crc, e.crc[part * L + l], (z_off_t)pb);
            }
        ok = ok && fwrite(e.crc.data(), 4, 2 * L, f) == 2 * L;
        crc = crc32(crc, reinterpret_cast<const Bytef*>(e.crc.data()), (uInt)(2 * L * 4));
        const uint32_t c32 = (uint32_t)crc;
        ok = ok && fwrite(&c32, 4, 1, f) == 1;
        ok = (fclose(f) == 0) && ok;
        MPIC_REQUIRE(ok && rename((path + ".tmp").c_str(), path.c_str()) == 0, MPIC_ERR_IO,
                     "failed to write " + path);
    }

    // demote_one_locked (cache.cpp:426-445): the least recently used entry of `from` goes
    // one tier down (Host -> Disk drops it when there is no disk tier).
    void demote(StoreKey key, StoreEntry& e, int to) {
        if (e.tier == MPIC_TIER_DEVICE && to >= MPIC_TIER_HOST) {
            const size_t pb = plane_bytes(e.T) * cfg.n_layers;
            MPIC_CUDA(cudaMallocHost(&e.hk, pb));
            MPIC_CUDA(cudaMallocHost(&e.hv, pb));
            void *k, *v;
            check_rc(mpic_kv_device_ptrs(e.kv, &k, &v));
            MPIC_CUDA(cudaMemcpyAsync(e.hk, k, pb, cudaMemcpyDeviceToHost, s));
            MPIC_CUDA(cudaMemcpyAsync(e.hv, v, pb, cudaMemcpyDeviceToHost, s));
            MPIC_CUDA(cudaStreamSynchronize(s));
            mpic_kv_free(e.kv);
            e.kv = nullptr;
            e.tier = MPIC_TIER_HOST;
        }
        if (e.tier == MPIC_TIER_HOST && to == MPIC_TIER_DISK) {
            if (!dir.empty()) write_file(key, e);
            cudaFreeHost(e.hk);
            cudaFreeHost(e.hv);
            e.hk = e.hv = nullptr;
            e.tier = MPIC_TIER_DISK;
            if (dir.empty()) index.erase(key);
        }
    }
    void enforce_budgets() {  // enforce_budgets_locked (cache.cpp:447-461)
        for (int from : {MPIC_TIER_DEVICE, MPIC_TIER_HOST}) {
            const uint32_t budget = from == MPIC_TIER_DEVICE ? device_budget : host_budget;
            for (;;) {
                uint32_t n = 0;
                auto victim = index.end();
                for (auto it = index.begin(); it != index.end(); ++it)
                    if (it->second.tier == from) {
                        ++n;
                        if (victim == index.end() || it->second.last_use < victim->second.last_use) victim = it;
                    }
                if (n <= budget) break;
                demote(victim->first, victim->second, from + 1);
            }
        }
    }

    // The entry as a Device-tier tensor (fetch, cache.cpp:261-304), or nullptr when a Host /
    // Disk copy fails its check on the device (the entry is then dropped).
    mpic_kv_t promote(const StoreKey& key, StoreEntry& e) {
        if (e.tier == MPIC_TIER_DEVICE) return e.kv;
        const uint32_t L = cfg.n_layers;
        const size_t pb = plane_bytes(e.T);
        mpic_kv_t kv = nullptr;
        check_rc(mpic_kv_alloc(L, e.T, cfg.n_heads, cfg.head_dim, dtype, device, &kv));
        void *k, *v;
        check_rc(mpic_kv_device_ptrs(kv, &k, &v));
        bool ok = true;
        std::vector<uint32_t> want = e.crc;
        if (e.tier == MPIC_TIER_HOST) {
            MPIC_CUDA(cudaMemcpyAsync(k, e.hk, pb * L, cudaMemcpyHostToDevice, s));
            MPIC_CUDA(cudaMemcpyAsync(v, e.hv, pb * L, cudaMemcpyHostToDevice, s));
        } else {  // Disk: header checks as open_mpic / deserialize_entry (cache.cpp:127-176)
            const std::string path = path_for(key);
            const int fd = open(path.c_str(), O_RDONLY);
            ok = fd >= 0;
            uint8_t h[84];
            struct stat st;
            const size_t want_size = 84 + 2 * pb * L + 8 * L + 4;
            ok = ok && fstat(fd, &st) == 0 && (size_t)st.st_size == want_size && pread(fd, h, 84, 0) == 84;
            uint32_t ver = 0, dims[5] = {};
            uint64_t fp = 0;
            if (ok) {
                std::memcpy(&ver, h + 4, 4);
                std::memcpy(&fp, h + 8, 8);
                std::memcpy(dims, h + 56, 20);
                ok = std::memcmp(h, "MPIC", 4) == 0 && ver == 3 && fp == mpic_config_fingerprint(&cfg) &&
                     std::memcmp(h + 24, key.hash.data(), 32) == 0 && dims[1] == L && dims[2] == e.T &&
                     dims[3] == cfg.n_heads && dims[4] == cfg.head_dim && h[76] == (dtype == MPIC_BF16 ? 1 : 0);
            }
            if (ok) {
                want.resize(2 * L);
                ok = pread(fd, want.data(), 8 * L, (off_t)(84 + 2 * pb * L)) == (ssize_t)(8 * L);
                e.position_base = dims[0];
            }
            void* pin = nullptr;
            if (ok) MPIC_CUDA(cudaMallocHost(&pin, pb * L));
            for (int part = 0; part < 2 && ok; ++part) {
                size_t got = 0;
                while (ok && got < pb * L) {
                    const ssize_t r = pread(fd, static_cast<char*>(pin) + got, std::min<size_t>(pb * L - got, 1u << 30),
                                            (off_t)(84 + part * pb * L + got));
                    ok = r > 0;
                    got += ok ? (size_t)r : 0;
                }
                if (ok) {
                    MPIC_CUDA(cudaMemcpyAsync(part ? v : k, pin, pb * L, cudaMemcpyHostToDevice, s));
                    MPIC_CUDA(cudaStreamSynchronize(s));  // the pinned slot is reused for V
                }
            }
            if (pin) cudaFreeHost(pin);
            if (fd >= 0) close(fd);
        }
        // the bytes are verified on the device, after the copy and before any use
        if (ok) ok = kv_crcs(kv, e.T) == want;
        if (!ok) {
            mpic_kv_free(kv);
            free_entry(e);
            if (e.tier == MPIC_TIER_DISK && !dir.empty()) unlink(path_for(key).c_str());
            index.erase(key);
            return nullptr;
        }
        free_entry(e);
        e.kv = kv;
        e.crc = want;
        e.tier = MPIC_TIER_DEVICE;
        return kv;
    }

    // compute_entry (transfer.cpp:41-58): prefill of the image's token ids at position base 0.
    mpic_kv_t compute(const uint8_t* hash32, uint32_t T) {
        if (!aux || aux_rows < T) {
            if (aux) mpic_workspace_destroy(aux);
            aux = nullptr;
            check_rc(mpic_workspace_create(model, T, T, &aux));
            aux_rows = T;
        }
        std::vector<int32_t> ids(T);
        check_rc(mpic_image_token_ids(&cfg, hash32, T, ids.data()));
        mpic_kv_t kv = nullptr;
        check_rc(mpic_kv_alloc(cfg.n_layers, T, cfg.n_heads, cfg.head_dim, dtype, device, &kv));
        std::vector<float> logits(cfg.vocab_size);
        const int rc = mpic_prefill_extend(model, aux, ids.data(), T, 0, 0, kv, logits.data(), s);
        if (rc != MPIC_OK) {
            mpic_kv_free(kv);
            check_rc(rc);
        }
        return kv;
    }
};

namespace {
StoreKey make_key(const uint8_t* hash32, const char* ns) {
    StoreKey k;
    std::memcpy(k.hash.data(), hash32, 32);
    k.ns = ns ? ns : "";
    return k;
}
}  // namespace

#define STORE_BEGIN try {
#define STORE_END                                   \
    return MPIC_OK;                                 \
    }                                               \
    catch (const mpicb::Error& e) {                 \
        mpicb::set_last_error(e.what());            \
        return e.code;                              \
    }                                               \
    catch (const std::exception& e) {               \
        mpicb::set_last_error(e.what());            \
        return MPIC_ERR_CUDA;                       \
    }

int mpic_store_create(mpic_model_t model, const char* dir, uint32_t device_budget, uint32_t host_budget,
                      mpic_store_t* out) {
    STORE_BEGIN
    MPIC_REQUIRE(model && out, MPIC_ERR_VALIDATION, "null model or output");
    auto st = std::make_unique<mpic_store_s>();
    st->model = model;
    check_rc(mpic_model_config_get(model, &st->cfg));
    st->dtype = mpic_model_dtype(model);
    st->device = mpic_model_device(model);
    st->dir = dir ? dir : "";
    while (st->dir.size() > 1 && st->dir.back() == '/') st->dir.pop_back();
    st->device_budget = device_budget;
    st->host_budget = host_budget;
    MPIC_CUDA(cudaSetDevice(st->device));
    MPIC_CUDA(cudaStreamCreateWithFlags(&st->s, cudaStreamNonBlocking));
    *out = st.release();
    STORE_END
}

int mpic_store_destroy(mpic_store_t store) {
    STORE_BEGIN
    if (!store) return MPIC_OK;
    cudaSetDevice(store->device);
    for (auto& kv : store->index) store->free_entry(kv.second);
    if (store->aux) mpic_workspace_destroy(store->aux);
    cudaStreamDestroy(store->s);
    delete store;
    STORE_END
}

int mpic_store_put(mpic_store_t store, const uint8_t* hash32, const char* ns, mpic_kv_t kv, uint32_t position_base) {
    STORE_BEGIN
    MPIC_REQUIRE(store && hash32 && kv, MPIC_ERR_VALIDATION, "null store, hash or kv");
    std::lock_guard<std::mutex> lk(store->mu);
    MPIC_CUDA(cudaSetDevice(store->device));
    uint32_t shape[4];
    mpic_dtype dt;
    check_rc(mpic_kv_shape(kv, shape, &dt));
    const mpic_model_config& c = store->cfg;
    MPIC_REQUIRE(shape[0] == c.n_layers && shape[2] == c.n_heads && shape[3] == c.head_dim, MPIC_ERR_VALIDATION,
                 "entry tensor shape does not match model");
    const uint32_t T = shape[1];
    mpic_kv_t own = nullptr;
    check_rc(mpic_kv_alloc(c.n_layers, T, c.n_heads, c.head_dim, store->dtype, store->device, &own));
    void *sk, *sv, *dk, *dv;
    check_rc(mpic_kv_device_ptrs(kv, &sk, &sv));
    check_rc(mpic_kv_device_ptrs(own, &dk, &dv));
    const size_t n = (size_t)c.n_layers * T * c.hidden_dim;
    if (dt == store->dtype) {
        MPIC_CUDA(cudaMemcpyAsync(dk, sk, n * elt_size(dt), cudaMemcpyDeviceToDevice, store->s));
        MPIC_CUDA(cudaMemcpyAsync(dv, sv, n * elt_size(dt), cudaMemcpyDeviceToDevice, store->s));
    } else if (dt == MPIC_F32) {
        launch_f32_to_bf16(static_cast<const float*>(sk), static_cast<__nv_bfloat16*>(dk), n, store->s);
        launch_f32_to_bf16(static_cast<const float*>(sv), static_cast<__nv_bfloat16*>(dv), n, store->s);
    } else {
        launch_bf16_to_f32(static_cast<const __nv_bfloat16*>(sk), static_cast<float*>(dk), n, store->s);
        launch_bf16_to_f32(static_cast<const __nv_bfloat16*>(sv), static_cast<float*>(dv), n, store->s);
    }
    StoreEntry e;
    e.kv = own;
    e.T = T;
    e.position_base = position_base;
    e.crc = store->kv_crcs(own, T);
    e.last_use = ++store->counter;
    const StoreKey key = make_key(hash32, ns);
    auto it = store->index.find(key);
    if (it != store->index.end()) {
        if (it->second.tier == MPIC_TIER_DISK && !store->dir.empty()) unlink(store->path_for(key).c_str());
        store->free_entry(it->second);
        store->index.erase(it);
    }
    store->index.emplace(key, std::move(e));
    store->enforce_budgets();
    STORE_END
}

int mpic_store_tier(mpic_store_t store, const uint8_t* hash32, const char* ns, int* tier) {
    STORE_BEGIN
    MPIC_REQUIRE(store && hash32 && tier, MPIC_ERR_VALIDATION, "null argument");
    std::lock_guard<std::mutex> lk(store->mu);
    const auto it = store->index.find(make_key(hash32, ns));
    *tier = it == store->index.end() ? -1 : it->second.tier;
    STORE_END
}

int mpic_store_demote(mpic_store_t store, const uint8_t* hash32, const char* ns, int tier) {
    STORE_BEGIN
    MPIC_REQUIRE(store && hash32, MPIC_ERR_VALIDATION, "null argument");
    MPIC_REQUIRE(tier >= MPIC_TIER_HOST && tier <= MPIC_TIER_DISK, MPIC_ERR_VALIDATION, "bad tier");
    std::lock_guard<std::mutex> lk(store->mu);
    MPIC_CUDA(cudaSetDevice(store->device));
    const StoreKey key = make_key(hash32, ns);
    auto it = store->index.find(key);
    MPIC_REQUIRE(it != store->index.end(), MPIC_ERR_NOT_FOUND, "cache entry not found: " + hex_of(hash32, 32));
    if (it->second.tier < tier) store->demote(key, it->second, tier);
    STORE_END
}

int mpic_store_remove(mpic_store_t store, const uint8_t* hash32, const char* ns) {
    STORE_BEGIN
    MPIC_REQUIRE(store && hash32, MPIC_ERR_VALIDATION, "null argument");
    std::lock_guard<std::mutex> lk(store->mu);
    const StoreKey key = make_key(hash32, ns);
    auto it = store->index.find(key);
    MPIC_REQUIRE(it != store->index.end(), MPIC_ERR_NOT_FOUND, "cache entry not found: " + hex_of(hash32, 32));
    if (it->second.tier == MPIC_TIER_DISK && !store->dir.empty()) unlink(store->path_for(key).c_str());
    store->free_entry(it->second);
    store->index.erase(it);
    STORE_END
}

int mpic_store_request(mpic_store_t store, mpic_workspace_t ws, const mpic_prompt* prompt, const mpic_policy* policy,
                       const char* ns, mpic_reposition reposition, mpic_kv_t linked, float* logits,
                       uint32_t* selected, uint32_t* m_out, uint32_t* chunk_status, void* stream) {
    STORE_BEGIN
    MPIC_REQUIRE(store && ws && prompt && policy, MPIC_ERR_VALIDATION, "null argument");
    std::lock_guard<std::mutex> lk(store->mu);
    MPIC_CUDA(cudaSetDevice(store->device));
    std::vector<mpic_kv_t> chunks;
    std::vector<uint32_t> bases, status;
    std::vector<StoreKey> used;
    std::vector<mpic_kv_t> computed_tmp;  // chunks computed for keys that could not be stored
    uint32_t img = 0;
    for (uint32_t sg = 0; sg < prompt->n_segments; ++sg) {
        if (prompt->kinds[sg] != 1) continue;
        const uint8_t* hash = prompt->hashes + 32 * (size_t)img++;
        const uint32_t T = prompt->lens[sg];
        const StoreKey key = make_key(hash, ns);
        mpic_kv_t kv = nullptr;
        uint32_t st = MPIC_CHUNK_LOADED;
        auto it = store->index.find(key);
        if (it != store->index.end() && it->second.T != T) {
            // token_count mismatch for the image segment (linker.cpp:281-285) is a link error
            throw Error(MPIC_ERR_LINK, "token_count mismatch for image segment");
        }
        if (it != store->index.end()) {
            kv = store->promote(key, it->second);
            if (!kv) st = MPIC_CHUNK_FALLBACK;
        } else {
            st = MPIC_CHUNK_COMPUTED;
        }
        if (!kv) {  // miss or fallback: compute the chunk and keep it (put, transfer.cpp:128-140)
            kv = store->compute(hash, T);
            StoreEntry e;
            e.kv = kv;
            e.T = T;
            e.position_base = 0;
            e.crc = store->kv_crcs(kv, T);
            store->index[key] = std::move(e);
        }
        StoreEntry& e = store->index.at(key);
        e.last_use = ++store->counter;
        chunks.push_back(kv);
        bases.push_back(e.position_base);
        status.push_back(st);
        used.push_back(key);
    }
    const int rc = mpic_request_prefill(store->model, ws, prompt, policy, chunks.data(), reposition, bases.data(),
                                        linked, logits, selected, m_out, stream);
    // budgets after the request: every chunk of the request stays resident while it runs
    store->enforce_budgets();
    check_rc(rc);
    if (chunk_status) std::memcpy(chunk_status, status.data(), status.size() * 4);
    STORE_END
}

int mpic_crc32_device(const void* d_ptr, size_t n, uint32_t* crc, void* stream) {
    STORE_BEGIN
    MPIC_REQUIRE(crc && (d_ptr || !n), MPIC_ERR_VALIDATION, "null argument");
    *crc = device_plane_crcs(d_ptr, n, 1, (cudaStream_t)stream)[0];
    STORE_END
}

int mpic_crc32_planes_device(const void* d_ptr, size_t plane_bytes, uint32_t n_planes, uint32_t* crcs, void* stream) {
    STORE_BEGIN
    MPIC_REQUIRE(crcs && (d_ptr || !plane_bytes || !n_planes), MPIC_ERR_VALIDATION, "null argument");
    constexpr uint32_t piece = 32 * 4096;  // the files loader's pieces
    const size_t ppp = (plane_bytes + piece - 1) / piece;
    if (!ppp || !n_planes) {
        for (uint32_t i = 0; i < n_planes; ++i) crcs[i] = (uint32_t)crc32(0L, Z_NULL, 0);
        return MPIC_OK;
    }
    cudaStream_t s = (cudaStream_t)stream;
    uint32_t* d = nullptr;
    MPIC_CUDA(cudaMallocAsync((void**)&d, ppp * n_planes * 4, s));
    launch_crc32_pieces(d_ptr, plane_bytes, n_planes, piece, d, s);
    std::vector<uint32_t> h(ppp * n_planes);
    MPIC_CUDA(cudaMemcpyAsync(h.data(), d, h.size() * 4, cudaMemcpyDeviceToHost, s));
    MPIC_CUDA(cudaFreeAsync(d, s));
    MPIC_CUDA(cudaStreamSynchronize(s));
    for (uint32_t i = 0; i < n_planes; ++i) crcs[i] = combine_crc_pieces(h.data() + i * ppp, plane_bytes, piece);
    STORE_END
}
