/* mpic_oracle — plain-C CPU restatement of the MPIC partial-reuse prefill path.
 *
 * TEST INFRASTRUCTURE ONLY. This is the checker: tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg may call it; the product (paper_2502_01960_b200)
 * never links or calls it.
 *
 * Parity pinned: tests/test_oracle.py checks every function here against the
 * unmodified reference built from source (oracle/_ref/libmpic_ref.so) and against
 * the committed golden fixtures in tests/golden/ (generated from that build by
 * oracle/gen_golden.py). Integer outputs are bit-exact; float outputs match the
 * reference within 1e-5 max-abs at the reference's own test shapes (dot products
 * here accumulate in double, OpenBLAS in float; every other rounding point — RoPE,
 * GELU, softmax, residual adds — is the reference's, in float).
 */
#ifndef MPIC_ORACLE_H
#define MPIC_ORACLE_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    uint32_t n_layers, n_heads, head_dim, hidden_dim, vocab_size, image_token_count;
    float rope_base;
    uint64_t seed;
} mo_config;

typedef struct {
    mo_config cfg;
    float* embedding; /* [V][h] */
    float* lm_head;   /* [V][h] */
    float** w;        /* per layer 6 matrices: wq wk wv wo [h][h], w1 [4h][h], w2 [h][4h] */
} mo_model;

uint64_t mo_fnv1a64(const uint8_t* bytes, size_t n);
uint64_t mo_fingerprint(const mo_config* c);
uint64_t mo_counter_hash(uint64_t seed, uint64_t stream, uint64_t i);
float mo_counter_uniform(uint64_t seed, uint64_t stream, uint64_t i);
uint32_t mo_crc32(const uint8_t* bytes, size_t n);

mo_model* mo_model_create(const mo_config* c);
void mo_model_free(mo_model* m);
float* mo_model_weight(mo_model* m, int which, uint32_t layer);

void mo_image_ids(const mo_config* c, const uint8_t* hash32, uint32_t count, int32_t* out);

/* Segments: kinds[s] 0=text 1=image, lens[s] tokens. policy 0=MpicK 1=TextOnly 2=All
 * 3=PrefixOnly. Returns |mask| (out must hold sum(lens) entries). */
uint32_t mo_select(uint32_t nseg, const uint8_t* kinds, const uint32_t* lens, int policy,
                   uint32_t k, int global, uint32_t* out);

/* Assembly: for image segment s (in order) chunk_k[i]/chunk_v[i] hold [L][len][h] and
 * chunk_base[i] its position_base. out_k/out_v [L][n][h] are fully written (text
 * slots zero). */
void mo_assemble(const mo_config* c, uint32_t nseg, const uint8_t* kinds, const uint32_t* lens,
                 const float* const* chunk_k, const float* const* chunk_v,
                 const uint32_t* chunk_base, int rerotate, float* out_k, float* out_v);

/* Selective pass: rows[i] ascending cache rows recomputed, token ids[i] (already
 * gathered), rotary position rope_pos[i]; each row attends over cache rows
 * [0, rows[i]]. kv [L][n_ctx][h] in/out. logits [V] of the last row. */
int mo_selective_core(const mo_model* m, const int32_t* ids, const uint32_t* rows,
                      const uint32_t* rope_pos, uint32_t cnt, float* kv_k, float* kv_v,
                      uint32_t n_ctx, float* logits);

#ifdef __cplusplus
}
#endif
#endif
