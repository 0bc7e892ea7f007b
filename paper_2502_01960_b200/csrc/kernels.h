// Internal kernel launchers of the MPIC B200 library (not part of the C ABI).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "mpic_b200.h"

namespace mpicb {

enum EpiMode : int { EPI_STORE = 0, EPI_QKV = 1, EPI_RESID = 2, EPI_GELU = 3, EPI_STORE_F32 = 4 };

// Fused GEMM epilogue description (shared by the SIMT and tcgen05 GEMMs).
struct EpiParams {
    int mode = EPI_STORE;
    // EPI_QKV: columns [0,h) -> q (rotated), [h,2h) -> kv_k[kv_rows[r]] (rotated),
    // [2h,3h) -> kv_v[kv_rows[r]]. kv_k/kv_v point at the layer's plane.
    void* q = nullptr;
    void* kv_k = nullptr;
    void* kv_v = nullptr;
    const uint32_t* kv_rows = nullptr;
    const uint32_t* rope_pos = nullptr;
    const float2* rope = nullptr;  // [pos][head_dim/2] (cos, sin)
    const float2* rope_tok = nullptr;  // optional [row][head_dim/2] (cos, sin) at rope_pos[row]
    uint32_t hidden = 0;
    uint32_t head_dim = 0;
    // EPI_RESID: x[row][col] += acc, and xb = bf16(x) when xb != null. The tcgen05 GEMM
    // may split K: partials go to `partial` ([split][rows_total][ldx] fp32, capacity
    // partial_cap floats) and a reduction kernel adds them (deterministic order).
    float* x = nullptr;
    __nv_bfloat16* xb = nullptr;
    uint32_t ldx = 0;
    uint32_t split_k = 1;
    float* partial = nullptr;
    size_t partial_cap = 0;
    uint32_t rows_total = 0;
    // EPI_STORE / EPI_GELU
    void* out = nullptr;
    uint32_t ldo = 0;
    uint32_t dbg = 0;  // pair GEMM diagnostics (MPIC_PG_DBG bits 16/32: skip x loads / stores)
};

// One chunk placement for the assembly kernel (device-side descriptor).
int hot_priority();  // launch priority of the hot kernels (capi.cu)

struct AsmChunk {
    const void* src_k;
    const void* src_v;
    uint32_t src_tokens;  // T of the source planes
    uint32_t src_row0;
    uint32_t dst_row0;
    uint32_t rows;
    uint32_t table;  // index of this chunk's (cos,sin) table in the rerotate tables
    uint32_t rotate; // 1 when this chunk's K rows are rotated
    uint32_t src_ld;   // elements per source row (the chunk's H*D); the destination row is H_dst*D
    uint32_t src_col0; // first source column copied (head-parallel: head0 * D)
};

void set_last_error(const std::string& m);  // the message mpic_last_error() returns

void launch_embed(const float* emb, const int32_t* ids, uint32_t m, uint32_t h, float* x,
                  __nv_bfloat16* xb, cudaStream_t s);
// out[i][j] = tab[pos[i]][j] for i < m, j < half_d (per-request RoPE rows).
void launch_rope_gather(const float2* tab, const uint32_t* pos, uint32_t m, uint32_t half_d, float2* out,
                        cudaStream_t s);
void launch_rope_table(const double* inv_freq, uint32_t half_d, uint32_t p0, uint32_t p1,
                       float2* tab, cudaStream_t s);
void launch_gemm_simt(const void* A, mpic_dtype a_t, uint32_t lda, const void* W, mpic_dtype w_t,
                      uint32_t M, uint32_t N, uint32_t K, const EpiParams& ep, mpic_dtype o_t,
                      cudaStream_t s);
// scratch (optional, fp32 head_dim 128): room for key-split partials (split x m x (h + 2H)
// floats); without it the fp32 attention runs unsplit.
void launch_attn_simt(const void* q, const void* k, const void* v, mpic_dtype dt,
                      const uint32_t* rows, uint32_t m, uint32_t H, uint32_t D, void* out,
                      cudaStream_t s, float* capture = nullptr, uint32_t T = 0, float* scratch = nullptr,
                      size_t scratch_floats = 0);
void launch_lm_head(const float* x_last, const void* W, mpic_dtype w_t, uint32_t V, uint32_t h,
                    float* logits, cudaStream_t s);
// out_k/out_v[l][i][:] = k/v[l][rows[i]][:] as fp32 (rows of a [L][T][h] cache).
void launch_gather_rows(const void* k, const void* v, mpic_dtype dt, uint32_t L, uint32_t T, uint32_t h,
                        const uint32_t* rows, uint32_t n_rows, float* out_k, float* out_v, cudaStream_t s);
void launch_clock_probe(float* out_mhz, uint32_t spin_ns, cudaStream_t s);
void launch_f32_to_bf16(const float* in, __nv_bfloat16* out, size_t n, cudaStream_t s);
void launch_bf16_to_f32(const __nv_bfloat16* in, float* out, size_t n, cudaStream_t s);
void launch_x_to_bf16(const float* x, __nv_bfloat16* xb, uint32_t m, uint32_t h, cudaStream_t s);

// Weight synthesis (model.cpp:28-36): dst[i] = counter_uniform(seed, (tag<<32)|layer, i)*scale
void launch_synth(uint64_t seed, uint64_t tag, uint32_t layer, size_t count, float scale,
                  void* dst, mpic_dtype dt, cudaStream_t s);
// Sub-matrix of the same synthetic weight: dst[r][j] = w[(row0 + r) * cols_total + col0 + j]
// for r < rows, j < ncols (head-parallel slices, bit-identical to the full matrix).
void launch_synth_2d(uint64_t seed, uint64_t tag, uint32_t layer, uint32_t rows, uint32_t cols_total,
                     uint32_t row0, uint32_t col0, uint32_t ncols, float scale, void* dst, mpic_dtype dt,
                     cudaStream_t s);
// x[i] += add[i], xb[i] = bf16(x[i]) over n floats (head-parallel reduce-scatter result).
void launch_resid_add(float* x, const float* add, __nv_bfloat16* xb, size_t n, cudaStream_t s);

// Chunk gather + optional K rerotation + dtype cast + gap zero-fill (linker.cpp:260-314).
void launch_assemble(const AsmChunk* d_chunks, uint32_t n_chunks, const float2* d_tables,
                     uint32_t n_tables, mpic_dtype src_t, void* dst_k, void* dst_v,
                     mpic_dtype dst_t, uint32_t L, uint32_t T_dst, uint32_t H, uint32_t D,
                     int zero_gaps, cudaStream_t s, uint32_t src_l0 = 0,
                     const uint8_t* skip_blk = nullptr);

// Attention work plan (tc_attn.cu): an item is up to two query tiles of one head that
// stream the same key blocks [b0, max(b1)) — tile[1] == kNoTile when the item has one.
constexpr uint32_t kNoTile = 0xffffffffu;
struct AttnUnit {
    uint32_t head, b0;
    uint32_t tile[2];
    uint32_t b1[2];    // per-tile end block
    uint32_t slot[2];  // kNoTile: write the final output; else partial slot for the combine
    uint32_t job[2];   // with a partial slot: its combine job (the last split to finish merges it)
};
struct AttnCombine {
    uint32_t tile, head, slot0, n;
};
struct AttnPlan {
    // units[0, items): the work items grouped by persistent CTA (CTA c runs items
    // [off[c], off[c + 1])), then the offsets themselves packed into the trailing entries
    // (attn_cta_offsets): one device buffer carries both
    std::vector<AttnUnit> units;
    std::vector<AttnCombine> combine;
    uint32_t slots = 0;
    uint32_t items = 0;
};
// The per-CTA item offsets stored after a plan's `items` work items.
#ifdef __CUDACC__
__host__ __device__
#endif
inline const uint32_t* attn_cta_offsets(const AttnUnit* units, uint32_t items) {
    return reinterpret_cast<const uint32_t*>(units + items);
}
unsigned long long* attn_debug_buffer();
// starts (optional, batched requests): per selected row, the first cache row of its request.
AttnPlan plan_attention(const uint32_t* rows, uint32_t m, uint32_t n_heads, const uint32_t* starts = nullptr);
// Query tiles are right-aligned: tile t holds selected rows [128t - shift, 128(t+1) - shift)
// with shift = 128 * ceil(m / 128) - m, so only the FIRST tile is partial. Rows are sorted by
// position, so every tile then ends at an earlier (or the same) row than with left-aligned
// tiles and needs at most as many key blocks (config C: 149 -> 130 tile-blocks per head).
inline uint32_t attn_tile_shift(uint32_t m) { return (m + 127) / 128 * 128 - m; }
inline uint32_t attn_tile_last_row(uint32_t t, uint32_t m) { return (t + 1) * 128 - attn_tile_shift(m) - 1; }
// Linking inside attention (device-resident bf16 chunks, no re-rotation): 128-key blocks
// that lie inside one cached chunk and hold no recomputed row are read by the attention
// kernel straight from the chunk's [L][T_c][h] planes, and the CTA that owns the block for
// the lowest query tile that reaches it stores it into the request cache (TMA store of the tile it already
// holds in shared memory). Every other block is assembled beforehand as usual. Lives in
// device memory, 64-B aligned; the per-block table follows the header.
constexpr uint32_t kMaxLinkChunks = 8;
constexpr uint32_t kLinkedBlock = 0xffffffffu;  // block read from the request cache
struct alignas(64) TmapBytes {
    unsigned char b[128];  // a CUtensorMap
};
struct alignas(64) AttnLink {
    TmapBytes maps[2 * kMaxLinkChunks];  // per chunk: K, V over [L * T_c rows][h]
    uint32_t tokens[kMaxLinkChunks];     // T_c
    uint32_t nblk;
    uint32_t pad[7];
    // uint32_t blk[nblk]: (chunk << 24) | first chunk row of the block, or kLinkedBlock
    // uint16_t wtile[nblk]: the query tile whose item stores block b (lowest tile reaching b)
};
void make_link_maps(AttnLink* host, const void* const* k, const void* const* v, const uint32_t* T, uint32_t n,
                    uint32_t L, uint32_t h);

void launch_attn_tc(const __nv_bfloat16* q, const __nv_bfloat16* kcache, const __nv_bfloat16* vcache,
                    uint32_t n_ctx, const uint32_t* d_rows, uint32_t m, uint32_t H,
                    const AttnUnit* d_units, uint32_t n_units, const AttnCombine* d_combine,
                    uint32_t n_combine, float* part_o, float2* part_ml, __nv_bfloat16* out,
                    cudaStream_t s, const AttnLink* link = nullptr, uint32_t layer = 0,
                    const uint32_t* d_starts = nullptr, uint32_t* d_counters = nullptr);

// tcgen05 / TMA kernels (tc_gemm.cu, tc_attn.cu)
struct TcGemmPlan;
bool tc_gemm_supported(uint32_t M, uint32_t N, uint32_t K);
// w_blocked: W is stored in 16 KB tiles [N/128][K/64][128][64] (pgemm_weight_layout), so
// every TMA box of the weight stream is one contiguous DRAM burst.
void launch_gemm_tc(const __nv_bfloat16* A, uint32_t lda, const __nv_bfloat16* W, uint32_t M,
                    uint32_t N, uint32_t K, const EpiParams& ep, cudaStream_t s, bool w_blocked = false);
// Persistent CTA-pair stream-K GEMM (tc_pgemm.cu): N % 256 == 0, K % 64 == 0.
bool pgemm_supported(uint32_t M, uint32_t N, uint32_t K);
void launch_pgemm(const __nv_bfloat16* A, const __nv_bfloat16* W, uint32_t M, uint32_t N, uint32_t K,
                  const EpiParams& ep, cudaStream_t s, bool w_blocked = false);
// fp32 mode on the tensor cores (3xTF32): operands pre-split by launch_tf32_split, fp32
// epilogue outputs. N % 256 == 0, K % 32 == 0.
bool pgemm_x3_supported(uint32_t M, uint32_t N, uint32_t K);
void launch_pgemm_x3(const float* A_hi, const float* A_lo, const float* W_hi, const float* W_lo, uint32_t M,
                     uint32_t N, uint32_t K, const EpiParams& ep, cudaStream_t s);
// hi = tf32_rna(x), lo = tf32_rna(x - hi) over n floats (n % 4 == 0, 16-B aligned).
void launch_tf32_split(const float* x, float* hi, float* lo, size_t n, cudaStream_t s);
// zlib CRC32 of n_planes consecutive planes of plane_bytes bytes at a device address, one
// value per `piece` bytes of each plane into d_out (async; store.cu), and the host combination
// of one plane's piece CRCs (h[ceil(plane_bytes / piece)]) into the plane's CRC.
void launch_crc32_pieces(const void* base, size_t plane_bytes, uint32_t n_planes, uint32_t piece, uint32_t* d_out,
                         cudaStream_t s);
uint32_t combine_crc_pieces(const uint32_t* h, size_t plane_bytes, uint32_t piece);
// MPIC_PG_TS diagnostics of the last pair GEMM's CTA 0: 5 x %globaltimer ns (entry, after
// prologue, MMAs issued, epilogue done, exit), then clock64 cycles: producer waiting on
// empty slots / producer total / MMA issuer waiting on full slots / MMA issuer total.
void pgemm_timestamps(unsigned long long* out9);
// Row-major [N][K] bf16 <-> the blocked weight layout (N % 128 == 0, K % 64 == 0).
void launch_block_weights(const __nv_bfloat16* src, __nv_bfloat16* dst, uint32_t N, uint32_t K, bool to_blocked,
                          cudaStream_t s);

} // namespace mpicb
