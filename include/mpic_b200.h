/* mpic_b200.h — C ABI of the B200-native MPIC partial-reuse prefill path.
 *
 * This is the drop-in boundary: plain C types, plain pointers and sizes, explicit CUDA
 * streams (passed as void*, i.e. a cudaStream_t), no C++ or torch types, no exceptions.
 * The C++ host library (include/mpic/ headers, same API as the reference
 * proj/include/mpic headers) sits on top of it; a cgo / JNI / ctypes binding would bind
 * exactly these symbols.
 *
 * Every call returns an mpic_status; codes map 1:1 onto the reference's exception
 * classes (proj/include/mpic/errors.h:10-62). mpic_last_error() returns the message of
 * the calling thread's last failure.
 *
 * Layouts (reference proj/include/mpic/tensor.h:11-55): KV is [L][T][H][D] row-major,
 * keys stored post-RoPE; weights are row-major [out][in] and every projection is
 * y = x·Wᵀ (proj/src/linker.cpp:64-65).
 */
#ifndef MPIC_B200_H
#define MPIC_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    MPIC_OK = 0,
    MPIC_ERR_CONFIG = 1,     /* mpic::config_error */
    MPIC_ERR_VALIDATION = 2, /* mpic::validation_error */
    MPIC_ERR_STATE = 3,      /* mpic::state_error */
    MPIC_ERR_LINK = 4,       /* mpic::link_error */
    MPIC_ERR_CONTRACT = 5,   /* mpic::contract_error */
    MPIC_ERR_FORMAT = 6,     /* mpic::format_error */
    MPIC_ERR_INTEGRITY = 7,  /* mpic::integrity_error */
    MPIC_ERR_IO = 8,         /* mpic::io_error */
    MPIC_ERR_NOT_FOUND = 9,  /* mpic::not_found_error */
    MPIC_ERR_REQUEST = 10,   /* mpic::request_error */
    MPIC_ERR_CUDA = 20,      /* CUDA runtime failure (no reference equivalent) */
    MPIC_ERR_NO_DEVICE = 21  /* no sm_100 device: the path never falls back to the CPU */
} mpic_status;

typedef enum { MPIC_F32 = 0, MPIC_BF16 = 1 } mpic_dtype;

typedef enum { MPIC_AS_STORED = 0, MPIC_REROTATE = 1 } mpic_reposition; /* linker.h:81-88 */

/* mpic::ModelConfig (proj/include/mpic/config.h:7-24), same field order and meaning. */
typedef struct {
    uint32_t n_layers;
    uint32_t n_heads;
    uint32_t head_dim;
    uint32_t hidden_dim;
    uint32_t vocab_size;
    uint32_t image_token_count;
    float rope_base;
    uint64_t seed;
} mpic_model_config;

typedef struct mpic_model_s* mpic_model_t;         /* device-resident weights */
typedef struct mpic_kv_s* mpic_kv_t;               /* device KV tensor [L][T][H][D] */
typedef struct mpic_workspace_s* mpic_workspace_t; /* per-request scratch */

const char* mpic_last_error(void);
const char* mpic_version(void);

/* ModelConfig::validate / fingerprint (proj/src/config.cpp:12-47). */
int mpic_config_validate(const mpic_model_config* cfg);
uint64_t mpic_config_fingerprint(const mpic_model_config* cfg);

/* ---- model ---------------------------------------------------------------------- */
/* build_model (proj/src/model.cpp:103-123), synthesised ON DEVICE: every fp32 weight is
 * bit-identical to the reference's counter_uniform(seed, (tag<<32)|layer, i) * scale,
 * then rounded to nearest-even when dtype == MPIC_BF16. */
int mpic_model_create(const mpic_model_config* cfg, int device, mpic_dtype dtype,
                      mpic_model_t* out);
/* The same model from caller-provided host weights (mpic::Model, model.h:16-30):
 * layer_w holds 6 pointers per layer in the order wq, wk, wv, wo, w1, w2. */
int mpic_model_upload(const mpic_model_config* cfg, int device, mpic_dtype dtype,
                      const float* embedding, const float* lm_head,
                      const float* const* layer_w, mpic_model_t* out);
int mpic_model_destroy(mpic_model_t model);
int mpic_model_config_get(mpic_model_t model, mpic_model_config* out);
/* The model's device ordinal. */
int mpic_model_device(mpic_model_t model);
mpic_dtype mpic_model_dtype(mpic_model_t model);
/* Copy one weight matrix back to host fp32 (which: 0 emb, 1 lm_head, 2..7 wq wk wv wo
 * w1 w2). Test hook for the bit-exact synthesis check. */
int mpic_model_download_weight(mpic_model_t model, int which, uint32_t layer, float* out);

/* ---- KV tensors ------------------------------------------------------------------ */
int mpic_kv_alloc(uint32_t n_layers, uint32_t n_tokens, uint32_t n_heads, uint32_t head_dim,
                  mpic_dtype dtype, int device, mpic_kv_t* out);
int mpic_kv_free(mpic_kv_t kv);
int mpic_kv_shape(mpic_kv_t kv, uint32_t* shape4, mpic_dtype* dtype);
/* Device pointers of the K and V planes (each L*T*H*D elements of the kv dtype). */
int mpic_kv_device_ptrs(mpic_kv_t kv, void** k, void** v);
/* Host fp32 <-> device (converting to/from bf16 on the device when needed).
 * Synchronous on `stream`. */
int mpic_kv_upload(mpic_kv_t kv, const float* k, const float* v, void* stream);
int mpic_kv_download(mpic_kv_t kv, float* k, float* v, void* stream);
/* Download only cache rows rows[0..n_rows) of every layer into host k/v laid out as the
 * full [L][T][H*D] tensor (other rows untouched). Synchronous. */
int mpic_kv_download_rows(mpic_kv_t kv, const uint32_t* rows, uint32_t n_rows, float* k, float* v,
                          void* stream);
/* Zero-fill rows [row0, row0+rows) of every layer (async). */
int mpic_kv_zero_rows(mpic_kv_t kv, uint32_t row0, uint32_t rows, void* stream);

/* ---- assembly: assemble_linked_cache (proj/src/linker.cpp:260-314) ---------------- */
/* One cached chunk placed into the request cache: rows [src_row0, src_row0+rows) of
 * `src` go to rows [dst_row0, ...) of the destination, for every layer. Under
 * MPIC_REROTATE the K rows are rotated by delta = dst_row0 - (position_base + src_row0)
 * (model.cpp:64-83; the delta is the same for every row of a chunk). */
typedef struct {
    mpic_kv_t src;
    uint32_t src_row0;
    uint32_t dst_row0;
    uint32_t rows;
    uint32_t position_base; /* KvCacheEntry::position_base of the chunk */
} mpic_chunk_ref;

/* Gathers all chunks into dst in ONE launch (async on `stream`). When zero_gaps != 0,
 * every dst row not covered by a chunk is zero-filled (the reference's Dummy slots,
 * tensor.h:20-23). Source and destination dtypes may differ (fp32 chunks from a host
 * staging buffer into a bf16 request cache). */
int mpic_assemble(void* stream, const mpic_chunk_ref* chunks, uint32_t n_chunks, mpic_kv_t dst,
                  mpic_reposition reposition, float rope_base, int zero_gaps);
/* Same with raw device pointers for the sources (e.g. a pinned/H2D staging ring):
 * src_k[i]/src_v[i] point at [L][src_tokens[i]][H][D] planes of dtype src_dtype. */
int mpic_assemble_raw(void* stream, const void* const* src_k, const void* const* src_v,
                      const uint32_t* src_tokens, mpic_dtype src_dtype,
                      const mpic_chunk_ref* chunks, uint32_t n_chunks, mpic_kv_t dst,
                      mpic_reposition reposition, float rope_base, int zero_gaps);

/* ---- selective recompute --------------------------------------------------------- */
/* Scratch for up to max_rows recomputed rows over caches of up to max_ctx tokens. */
int mpic_workspace_create(mpic_model_t model, uint32_t max_rows, uint32_t max_ctx,
                          mpic_workspace_t* out);
int mpic_workspace_destroy(mpic_workspace_t ws);

/* selective_core (proj/src/linker.cpp:35-135): recompute Q/K/V and the full layer
 * stack for the `m` rows `rows` (ascending cache indices; token ids `ids`), rotate Q/K
 * at their own index, scatter K/V into `kv`, attend each row over kv rows [0, row],
 * and write the first-token logits (vocab floats) of the last row.
 * Host pointers; synchronous (returns when logits are in host memory). */
int mpic_selective_prefill(mpic_model_t model, mpic_workspace_t ws, const int32_t* ids,
                           const uint32_t* rows, uint32_t m, mpic_kv_t kv, float* logits,
                           void* stream);
/* extend_rows (proj/src/model.cpp:211-330): rows [start, start+m) of kv recomputed for
 * `ids` at rotary positions position_base+start+i. kv must already hold start+m rows. */
int mpic_prefill_extend(mpic_model_t model, mpic_workspace_t ws, const int32_t* ids, uint32_t m,
                        uint32_t start, uint32_t position_base, mpic_kv_t kv, float* logits,
                        void* stream);
/* General host form behind both: ids/rows/rope_pos are host arrays. Optional outputs:
 * hidden_out [m][hidden_dim] final-layer hidden rows (mean_pooled_hidden, model.cpp:369-389);
 * attn_capture [L][H][T][T] normalised attention of each recomputed row at query index
 * rows[i] (AttentionDump, model.h:50-71; fp32 models only; other rows left zero). */
int mpic_forward_rows(mpic_model_t model, mpic_workspace_t ws, const int32_t* ids,
                      const uint32_t* rows, const uint32_t* rope_pos, uint32_t m, mpic_kv_t kv,
                      float* logits, float* hidden_out, float* attn_capture, void* stream);
/* Layer-0 keys of `ids` rotated at `positions`, out [m][hidden_dim] fp32 (the CacheBlend
 * deviation probe, proj/src/linker.cpp:485-499). Synchronous. */
int mpic_layer0_keys(mpic_model_t model, mpic_workspace_t ws, const int32_t* ids,
                     const uint32_t* positions, uint32_t m, float* out, void* stream);
/* Fully asynchronous form of both: every pointer is a DEVICE pointer, ids are assumed
 * in-vocabulary (the host forms validate), max_pos >= every row and rotary position,
 * logits land in d_logits on `stream`. */
int mpic_forward_rows_async(mpic_model_t model, mpic_workspace_t ws, const int32_t* d_ids,
                            const uint32_t* d_rows, const uint32_t* d_rope_pos, uint32_t m,
                            uint32_t max_pos, mpic_kv_t kv, float* d_logits, void* stream);

/* ---- request-level host logic (integer work; bit-exact with the reference) -------- */
/* A segmented prompt (SegmentedPrompt, proj/include/mpic/linker.h:14-54) as flat arrays. */
typedef struct {
    uint32_t n_segments;
    const uint8_t* kinds;    /* per segment: 0 = text, 1 = image */
    const uint32_t* lens;    /* per segment token count */
    const int32_t* text_ids; /* text segments' ids, concatenated in order */
    const uint8_t* hashes;   /* 32-byte content hash per image segment, in order */
} mpic_prompt;

typedef enum {
    MPIC_POLICY_MPIC_K = 0, /* MpicKPolicy (linker.h:58-63) */
    MPIC_POLICY_TEXT_ONLY = 1,
    MPIC_POLICY_ALL = 2,
    MPIC_POLICY_PREFIX_ONLY = 3
} mpic_policy_tag;

typedef struct {
    int policy;        /* mpic_policy_tag */
    uint32_t k;        /* MpicKPolicy::k */
    int global_budget; /* MpicKPolicy::global */
} mpic_policy;

/* image_token_ids (proj/src/model.cpp:148-156). */
int mpic_image_token_ids(const mpic_model_config* cfg, const uint8_t* hash32, uint32_t count,
                         int32_t* out);
/* select_tokens (proj/src/linker.cpp:209-258): out holds total_tokens entries; *m = |mask|. */
int mpic_select_tokens(const mpic_prompt* prompt, const mpic_policy* policy, uint32_t* out,
                       uint32_t* m);
/* SegmentedPrompt::flatten_ids (proj/src/linker.cpp:160-172): out holds total_tokens ids. */
int mpic_flatten_ids(const mpic_model_config* cfg, const mpic_prompt* prompt, int32_t* out);

/* One MPIC-k request end to end on the device: select_tokens -> assemble_linked_cache ->
 * selective_prefill (the composition of test_transfer.cpp:153-188). chunks[i] is the
 * device-resident (Device tier) entry of the i-th image segment, position_bases[i] its
 * KvCacheEntry::position_base. `linked` receives the finished [L][n][H][D] cache;
 * `selected` (may be NULL; else n entries) the recompute set, *m_out its size; logits
 * (host, vocab floats) the first-token logits. Synchronous on `stream`. */
int mpic_request_prefill(mpic_model_t model, mpic_workspace_t ws, const mpic_prompt* prompt,
                         const mpic_policy* policy, const mpic_kv_t* chunks,
                         mpic_reposition reposition, const uint32_t* position_bases,
                         mpic_kv_t linked, float* logits, uint32_t* selected, uint32_t* m_out,
                         void* stream);
/* Same request with the chunk KV in HOST memory (fp32 [L][len][H][D] per image, pinned for
 * full PCIe rate): the loader streams layer l of every chunk to HBM on a side stream while
 * layer l-1 is being recomputed; each landed layer is assembled (and cast to the model
 * dtype) right before it is used. */
/* The same request with each image's chunk read from a .mpic file (paths[i] for the i-th
 * image segment; v1 fp32, v2 bf16, v3 = v2/v1 plus per-layer CRCs): reader threads pread
 * layer l of every chunk into a pinned ring slot while the GPU computes layer l-1, and the
 * copy stream moves the slot to HBM. position_base comes from each file's header.
 * Fault semantics of prepare (proj/src/transfer.cpp:83-145, cache.cpp:171-176): a NULL path
 * or a file that does not exist is a miss (MPIC_CHUNK_COMPUTED); a file with a bad header,
 * another model's fingerprint, the wrong shape or token count, a content hash other than
 * the prompt's image hash, a short read or a CRC mismatch is a fallback
 * (MPIC_CHUNK_FALLBACK). Either way the chunk is computed on the device (compute_entry,
 * transfer.cpp:41-58) on a side stream concurrently with the loads, and the request uses
 * it layer by layer. Every loaded layer is CRC-checked on the GPU right after its H2D (v3:
 * against the per-layer table; MPIC_FILES_CRC=host checks v3 layers on the reader threads
 * before the H2D instead); the per-layer and file CRCs are known
 * only after the last layer, and a mismatch re-runs the request with the chunk computed:
 * the outputs never come from a corrupt chunk. chunk_status (may be NULL) receives one
 * mpic_chunk_status per image segment. */
typedef enum { MPIC_CHUNK_LOADED = 0, MPIC_CHUNK_COMPUTED = 1, MPIC_CHUNK_FALLBACK = 2 } mpic_chunk_status;
int mpic_request_prefill_files2(mpic_model_t model, mpic_workspace_t ws, const mpic_prompt* prompt,
                                const mpic_policy* policy, const char* const* paths, mpic_reposition reposition,
                                mpic_kv_t linked, float* logits, uint32_t* selected, uint32_t* m_out,
                                uint32_t* chunk_status, void* stream);
/* mpic_request_prefill_files2 without the per-chunk report. */
int mpic_request_prefill_files(mpic_model_t model, mpic_workspace_t ws, const mpic_prompt* prompt,
                               const mpic_policy* policy, const char* const* paths, mpic_reposition reposition,
                               mpic_kv_t linked, float* logits, uint32_t* selected, uint32_t* m_out, void* stream);

/* Batched varlen MPIC-k: nreq independent requests (device-resident chunks,
 * request-major in `chunks`) in ONE selective pass on the bf16 head_dim-128 path. Request
 * r's cache occupies rows [off_r, off_r + n_r) of `linked` (off_r = sum of the earlier
 * prompts' lengths; linked->T >= sum n_r); its rows attend only to its own rows. logits:
 * [nreq][vocab] host floats; m_out[r] = rows recomputed for request r. Synchronous.
 * Replaces nreq calls of the reference's assemble_linked_cache + selective_prefill
 * (proj/include/mpic/linker.h:107-129), which has no batched form. */
int mpic_request_prefill_batch(mpic_model_t model, mpic_workspace_t ws, const mpic_prompt* prompts, uint32_t nreq,
                               const mpic_policy* policy, const mpic_kv_t* chunks, mpic_reposition reposition,
                               mpic_kv_t linked, float* logits, uint32_t* m_out, void* stream);

/* ---- head-parallel request (one long request over P GPUs) ---------------
 * Rank r owns heads [head0, head0 + n_local_heads): its model holds those heads' Wq/Wk/Wv
 * rows and Wo columns (bit-identical slices of build_model's weights) and the full FFN; its
 * request cache is [L][n][n_local_heads][D]. Per layer l the caller runs
 *   mpic_hp_layer_attn(l) -> partial[m_pad][h] (fp32: this rank's heads' share of attn.Wo^T)
 *   reduce-scatter(sum) of partial over the P ranks, rank r receiving rows [r*mr, (r+1)*mr)
 *   mpic_hp_layer_ffn(l, reduced, r*mr, mr) -> x/xb rows updated (residual + FFN)
 *   all-gather of the bf16 rows of xb (in place, mpic_workspace_device_ptr(ws, 1))
 * with m_pad = mr * P >= m. The rank holding row m-1 calls mpic_hp_logits(m-1). Partial
 * rows >= m must be zero. bf16 models with head_dim 128 only. */
int mpic_model_create_heads(const mpic_model_config* cfg, int device, mpic_dtype dtype, uint32_t head0,
                            uint32_t n_local_heads, mpic_model_t* out);
int mpic_hp_prepare(mpic_model_t model, mpic_workspace_t ws, const mpic_prompt* prompt, const mpic_policy* policy,
                    const mpic_kv_t* chunks, mpic_reposition reposition, const uint32_t* position_bases,
                    mpic_kv_t linked, uint32_t* selected, uint32_t* m_out, void* stream);
int mpic_hp_layer_attn(mpic_model_t model, mpic_workspace_t ws, uint32_t layer, mpic_kv_t linked, float* d_partial,
                       void* stream);
int mpic_hp_layer_ffn(mpic_model_t model, mpic_workspace_t ws, uint32_t layer, const float* d_reduced, uint32_t row0,
                      uint32_t rows, void* stream);
int mpic_hp_logits(mpic_model_t model, mpic_workspace_t ws, uint32_t row, float* logits, void* stream);
/* The whole head-parallel request on one rank, collectives inside the library: per layer
 * mpic_hp_layer_attn -> ncclReduceScatter(sum) of the Wo partials -> mpic_hp_layer_ffn on
 * this rank's rows -> in-place ncclAllGather of the bf16 rows; the owner of row m-1
 * computes the logits and broadcasts them, so every rank returns them. `nccl_comm` is an
 * ncclComm_t of P ranks whose rank r holds heads [r*H/P, (r+1)*H/P) (its model from
 * mpic_model_create_heads), or NULL for P = 1. The workspace needs max_rows >= m + P. With
 * graphs on (mpic_workspace_set_graphs) a request with the same shape as the previous one
 * records the layer loop — kernels and collectives — as one CUDA graph, replayed after
 * that. Replaces the per-head loop (linker.cpp:80-113) and the Wo reduction
 * (linker.cpp:115-118) of selective_prefill for one request split over P GPUs. */
int mpic_hp_request(mpic_model_t model, mpic_workspace_t ws, void* nccl_comm, const mpic_prompt* prompt,
                    const mpic_policy* policy, const mpic_kv_t* chunks, mpic_reposition reposition,
                    const uint32_t* position_bases, mpic_kv_t linked, float* logits, uint32_t* selected,
                    uint32_t* m_out, void* stream);
/* NCCL communicator plumbing for mpic_hp_request (libnccl.so.2 is loaded at run time):
 * rank 0 creates the id, the caller distributes its MPIC_NCCL_ID_BYTES bytes (any
 * out-of-band channel), every rank creates its communicator on its device. */
#define MPIC_NCCL_ID_BYTES 128
int mpic_nccl_unique_id(uint8_t* out);
int mpic_nccl_comm_create(const uint8_t* id, int nranks, int rank, int device, void** out);
int mpic_nccl_comm_destroy(void* comm);
/* Device pointer of a workspace buffer: 0 = x (fp32 [m_pad][h]), 1 = xb (bf16 [m_pad][h]). */
int mpic_workspace_device_ptr(mpic_workspace_t ws, int which, void** out);

/* CUDA-graph replay of mpic_request_prefill (default on): a request with the same launch
 * signature as the previous one on this workspace (model, linked cache, n, m, chunk count,
 * plan sizes) is captured once and replayed after that, with its inputs re-staged. */
int mpic_workspace_set_graphs(mpic_workspace_t ws, int on);

int mpic_request_prefill_host(mpic_model_t model, mpic_workspace_t ws, const mpic_prompt* prompt,
                              const mpic_policy* policy, const float* const* chunk_k,
                              const float* const* chunk_v, const uint32_t* position_bases,
                              mpic_reposition reposition, mpic_kv_t linked, float* logits,
                              uint32_t* selected, uint32_t* m_out, void* stream);
/* The same with the Host-tier chunks in `chunk_dtype` (MPIC_BF16: the model dtype, half the
 * PCIe bytes of the fp32 .mpic v1 payload). A NULL chunk_k[i] / chunk_v[i] is a miss: the
 * chunk is computed on the device (prefill of the image's token ids at position base 0,
 * transfer.cpp:41-58) on a side stream while the other chunks stream in, and its
 * position_bases entry is ignored (0). */
int mpic_request_prefill_host2(mpic_model_t model, mpic_workspace_t ws, const mpic_prompt* prompt,
                               const mpic_policy* policy, const void* const* chunk_k, const void* const* chunk_v,
                               mpic_dtype chunk_dtype, const uint32_t* position_bases, mpic_reposition reposition,
                               mpic_kv_t linked, float* logits, uint32_t* selected, uint32_t* m_out, void* stream);

/* ---- tiered chunk store on the device (CacheStore, proj/include/mpic/cache.h:70-133) ---
 * Entries are keyed by (content hash, namespace) for the store's model. Device tier: a KV
 * tensor in HBM in the model dtype; Host tier: pinned memory; Disk tier: a .mpic v3 file
 * under dir/<hex(ns)>/<fingerprint>/<hex(hash)>.mpic (cache.cpp:198-201; dir NULL or "" =
 * no disk tier: Host-tier victims are dropped). device_budget / host_budget are entry
 * counts; the least recently used entry beyond a budget moves one tier down
 * (cache.cpp:426-461). The per-layer CRC32s of every entry are computed on the GPU when it
 * enters the store and checked on the GPU after every Host / Disk -> Device promotion. */
typedef struct mpic_store_s* mpic_store_t;
typedef enum { MPIC_TIER_DEVICE = 0, MPIC_TIER_HOST = 1, MPIC_TIER_DISK = 2 } mpic_tier;
int mpic_store_create(mpic_model_t model, const char* dir, uint32_t device_budget, uint32_t host_budget,
                      mpic_store_t* out);
int mpic_store_destroy(mpic_store_t store);
/* put (cache.cpp:203-225): a copy of kv (cast to the model dtype) enters the Device tier. */
int mpic_store_put(mpic_store_t store, const uint8_t* hash32, const char* ns, mpic_kv_t kv, uint32_t position_base);
/* tier_of (cache.cpp:249-254): *tier = mpic_tier, or -1 when absent. */
int mpic_store_tier(mpic_store_t store, const uint8_t* hash32, const char* ns, int* tier);
/* demote_to (cache.cpp:363-380, test hook): move an entry down to `tier`. */
int mpic_store_demote(mpic_store_t store, const uint8_t* hash32, const char* ns, int tier);
int mpic_store_remove(mpic_store_t store, const uint8_t* hash32, const char* ns);
/* prepare + selective_prefill (transfer.cpp:83-145 with test_transfer.cpp:153-188): every image
 * chunk of the prompt is fetched into the Device tier (Host / Disk entries copied to HBM and
 * CRC-checked on the device); a miss, and an entry that fails its checks, is computed on the
 * device (compute_entry, transfer.cpp:41-58) and stored; then the device-resident MPIC request
 * runs (mpic_request_prefill). Budgets are enforced after the request. chunk_status (may be
 * NULL): one mpic_chunk_status per image segment. */
int mpic_store_request(mpic_store_t store, mpic_workspace_t ws, const mpic_prompt* prompt, const mpic_policy* policy,
                       const char* ns, mpic_reposition reposition, mpic_kv_t linked, float* logits,
                       uint32_t* selected, uint32_t* m_out, uint32_t* chunk_status, void* stream);
/* zlib-compatible CRC32 of n bytes of device memory (the store's GPU CRC). Synchronous. */
int mpic_crc32_device(const void* d_ptr, size_t n, uint32_t* crc, void* stream);
/* Per-plane CRC32s of n_planes consecutive planes of plane_bytes bytes of device memory, as
 * the disk loader computes them after each layer's H2D (128 KB pieces, one warp each for
 * plane_bytes % 4096 == 0, combined on the host). Synchronous. */
int mpic_crc32_planes_device(const void* d_ptr, size_t plane_bytes, uint32_t n_planes, uint32_t* crcs, void* stream);

/* Host-pointer fp32 GEMM on the device: c[M][N] = a[M][K] . b[N][K]^T (SIMT FFMA). Backs the
 * reference's gemm_nt/gemm_nn shims (proj/include/mpic/matmul.h:11-21). Synchronous. */
int mpic_host_gemm_f32(const float* a, const float* b, uint32_t M, uint32_t N, uint32_t K, float* c,
                       int device);

/* Pinned host memory for chunk staging (cudaMallocHost); mpic_host_free releases it. */
int mpic_host_alloc(size_t bytes, void** out);
int mpic_host_free(void* p);

/* Test hook: out[M][N] (fp32, device) = A[M][K] . W[N][K]^T for bf16 device operands,
 * through the tcgen05 GEMM (path 1), the tcgen05 GEMM on a blocked copy of W made on the
 * device (path 2), the tcgen05 GEMM with d_w already blocked [N/128][K/64][128][64]
 * (path 3) or the SIMT GEMM (path 0); for fp32 device operands, the fp32 mode's 3xTF32
 * tcgen05 GEMM (path 4, operands split on the device) or the SIMT FFMA GEMM (path 5).
 * Async on `stream`. */
int mpic_test_gemm(const void* d_a, const void* d_w, uint32_t M, uint32_t N, uint32_t K, int path,
                   float* d_out, void* stream);
/* Test hook: the tcgen05 GEMM with a fused epilogue. mode 0: residual (d_x fp32 [M][N]
 * += A.W^T, d_xb bf16 copy of the new x); mode 1: GELU (d_out bf16 [M][N]); mode 2: plain
 * bf16 store (d_out). Async on `stream`. */
int mpic_test_gemm_epi(const void* d_a, const void* d_w, uint32_t M, uint32_t N, uint32_t K, int mode,
                       float* d_x, void* d_xb, void* d_out, void* stream);

/* Test hook: the QKV projection exactly as a layer runs it (K3: the GEMM of the bf16 rows
 * d_a [M][K] with Wqkv d_w [3h][K], fused RoPE of q and k with the per-row (cos, sin)
 * table d_rope_tok [M][D/2] and the scatter of k, v to rows d_rows[i] of the bf16 cache
 * planes d_kv_k / d_kv_v [*][h]); q (rotated, bf16 [M][h]) -> d_q. Async on `stream`. */
int mpic_test_qkv(const void* d_a, const void* d_w, uint32_t M, uint32_t h, uint32_t K, uint32_t head_dim,
                  const uint32_t* d_rows, const void* d_rope_tok, void* d_q, void* d_kv_k, void* d_kv_v,
                  void* stream);

/* ---- per-phase device timing ------------------------------------------------------ */
typedef enum {
    MPIC_PHASE_ASSEMBLE = 0, /* K2 chunk gather (+ rerotate, cast) */
    MPIC_PHASE_EMBED = 1,
    MPIC_PHASE_QKV = 2,      /* K3 QKV GEMM + RoPE + KV scatter */
    MPIC_PHASE_ATTN = 3,     /* K4 selective attention */
    MPIC_PHASE_WO = 4,       /* K5 Wo GEMM + residual */
    MPIC_PHASE_W1 = 5,       /* K6 W1 GEMM + GELU */
    MPIC_PHASE_W2 = 6,       /* K7 W2 GEMM + residual */
    MPIC_PHASE_CAST = 7,     /* fp32 residual -> bf16 operand */
    MPIC_PHASE_LM_HEAD = 8,  /* K8 */
    MPIC_PHASE_COUNT = 9
} mpic_phase;
/* When enabled, every phase records CUDA events on its launching stream. collect()
 * waits for them and returns per-phase summed milliseconds and instance counts
 * (arrays of MPIC_PHASE_COUNT), then resets. */
int mpic_profile_enable(int on);
int mpic_profile_collect(double* ms, uint32_t* counts);

/* Test hook: the head_dim-128 tcgen05 selective attention on bf16 device buffers
 * q [m][H*128], k/v [n_ctx][H*128]; query i attends keys [0, rows[i]] (host rows,
 * ascending). out [m][H*128] bf16. Async on `stream`. */
/* Host-only inspection of the tcgen05 attention work plan (tc_attn.cu plan_attention) for
 * the recomputed rows' positions `rows` (ascending), m rows, n_heads heads, optional batched
 * request starts: counts[0] = work items, counts[1] = persistent CTAs, counts[2] = combine
 * jobs, counts[3] = partial slots. units_out (may be NULL, units_cap entries of 10 uint32:
 * head, b0, tile[2], b1[2], slot[2], job[2]) receives the items grouped by CTA, offs_out
 * (ctas + 1 entries) the per-CTA item offsets, jobs_out (4 uint32 each: tile, head, slot0,
 * n) the combine jobs. No GPU needed. Diagnostics / tests. */
int mpic_attention_plan(const uint32_t* rows, uint32_t m, uint32_t n_heads, const uint32_t* starts,
                        uint32_t* counts, uint32_t* units_out, uint32_t units_cap, uint32_t* offs_out,
                        uint32_t offs_cap, uint32_t* jobs_out, uint32_t jobs_cap);
int mpic_test_attention(const void* d_q, const void* d_k, const void* d_v, const uint32_t* rows,
                        uint32_t m, uint32_t n_ctx, uint32_t n_heads, void* d_out, void* stream);

/* Diagnostics: the SM clock (MHz) measured on the device — clock64 cycles over a
 * %globaltimer window of spin_ns — written to d_out_mhz. Async on `stream`. */
int mpic_clock_probe(float* d_out_mhz, uint32_t spin_ns, void* stream);

/* Number of kernels the last forward/assemble call on this thread launched. */
uint32_t mpic_last_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* MPIC_B200_H */
