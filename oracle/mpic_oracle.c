/* mpic_oracle.c — plain-C restatement of the reference's partial-reuse prefill path.
 * TEST INFRASTRUCTURE ONLY (see mpic_oracle.h). Compile with -ffp-contract=off so
 * float expressions round exactly where the reference's x86-64 build does.
 * Each function cites the reference file:line under /root/reference/proj it follows. */
#include "mpic_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* include/mpic/hash.h:18-25 */
uint64_t mo_fnv1a64(const uint8_t* bytes, size_t n) {
    uint64_t h = 0xcbf29ce484222325ull;
    for (size_t i = 0; i < n; ++i) {
        h ^= bytes[i];
        h *= 0x100000001b3ull;
    }
    return h;
}

/* src/config.cpp:30-47: FNV-1a over eight little-endian u64 fields, rope_base as its
 * f32 bit pattern. */
uint64_t mo_fingerprint(const mo_config* c) {
    uint64_t f[8];
    uint32_t rb;
    memcpy(&rb, &c->rope_base, 4);
    f[0] = c->n_layers; f[1] = c->n_heads; f[2] = c->head_dim; f[3] = c->hidden_dim;
    f[4] = c->vocab_size; f[5] = c->image_token_count; f[6] = rb; f[7] = c->seed;
    uint8_t buf[64];
    for (int j = 0; j < 8; ++j)
        for (int b = 0; b < 8; ++b) buf[8 * j + b] = (uint8_t)(f[j] >> (8 * b));
    return mo_fnv1a64(buf, 64);
}

/* include/mpic/rng.h:10-30 */
static uint64_t mix64(uint64_t x) {
    x ^= x >> 30;
    x *= 0xbf58476d1ce4e5b9ull;
    x ^= x >> 27;
    x *= 0x94d049bb133111ebull;
    x ^= x >> 31;
    return x;
}
uint64_t mo_counter_hash(uint64_t seed, uint64_t stream, uint64_t i) {
    const uint64_t phi = 0x9e3779b97f4a7c15ull;
    uint64_t h = mix64(seed + phi);
    h = mix64(h ^ (stream + phi));
    return mix64(h ^ (i + phi));
}
float mo_counter_uniform(uint64_t seed, uint64_t stream, uint64_t i) {
    const uint32_t bits = (uint32_t)(mo_counter_hash(seed, stream, i) >> 40);
    return (float)bits * (2.0f / 16777216.0f) - 1.0f;
}

/* zlib crc32 (reflected 0xEDB88320), as used by src/hash.cpp:58-62 */
uint32_t mo_crc32(const uint8_t* p, size_t n) {
    static uint32_t table[256];
    static int init = 0;
    if (!init) {
        for (uint32_t i = 0; i < 256; ++i) {
            uint32_t c = i;
            for (int k = 0; k < 8; ++k) c = (c & 1) ? 0xEDB88320u ^ (c >> 1) : c >> 1;
            table[i] = c;
        }
        init = 1;
    }
    uint32_t c = 0xFFFFFFFFu;
    for (size_t i = 0; i < n; ++i) c = table[(c ^ p[i]) & 0xff] ^ (c >> 8);
    return c ^ 0xFFFFFFFFu;
}

/* src/model.cpp:17-36, 103-123: counter-hash weight synthesis, stream (tag<<32)|layer */
static float* synth(uint64_t seed, uint64_t tag, uint32_t layer, size_t rows, size_t cols,
                    float scale) {
    float* w = (float*)malloc(rows * cols * sizeof(float));
    const uint64_t stream = (tag << 32) | layer;
    for (size_t i = 0; i < rows * cols; ++i) w[i] = mo_counter_uniform(seed, stream, i) * scale;
    return w;
}

mo_model* mo_model_create(const mo_config* c) {
    if (!c->n_layers || !c->n_heads || !c->head_dim || c->hidden_dim != c->n_heads * c->head_dim ||
        c->vocab_size < 2)
        return NULL;
    mo_model* m = (mo_model*)calloc(1, sizeof(mo_model));
    const size_t h = c->hidden_dim;
    const float scale = 1.0f / sqrtf((float)h);
    m->cfg = *c;
    m->embedding = synth(c->seed, 100, 0, c->vocab_size, h, 1.0f);
    m->lm_head = synth(c->seed, 101, 0, c->vocab_size, h, scale);
    m->w = (float**)calloc((size_t)6 * c->n_layers, sizeof(float*));
    for (uint32_t l = 0; l < c->n_layers; ++l) {
        m->w[6 * l + 0] = synth(c->seed, 1, l, h, h, scale);
        m->w[6 * l + 1] = synth(c->seed, 2, l, h, h, scale);
        m->w[6 * l + 2] = synth(c->seed, 3, l, h, h, scale);
        m->w[6 * l + 3] = synth(c->seed, 4, l, h, h, scale);
        m->w[6 * l + 4] = synth(c->seed, 5, l, 4 * h, h, scale);
        m->w[6 * l + 5] = synth(c->seed, 6, l, h, 4 * h, scale);
    }
    return m;
}

void mo_model_free(mo_model* m) {
    if (!m) return;
    for (uint32_t i = 0; i < 6 * m->cfg.n_layers; ++i) free(m->w[i]);
    free(m->w);
    free(m->embedding);
    free(m->lm_head);
    free(m);
}

/* which: 0 emb, 1 lm_head, 2..7 wq wk wv wo w1 w2 */
float* mo_model_weight(mo_model* m, int which, uint32_t layer) {
    if (which == 0) return m->embedding;
    if (which == 1) return m->lm_head;
    return m->w[6 * layer + (which - 2)];
}

/* src/model.cpp:148-156 */
void mo_image_ids(const mo_config* c, const uint8_t* hash32, uint32_t count, int32_t* out) {
    const uint64_t key = mo_fnv1a64(hash32, 32) ^ mo_fingerprint(c);
    for (uint32_t i = 0; i < count; ++i)
        out[i] = (int32_t)(mo_counter_hash(key, 0x696d67, i) % c->vocab_size);
}

/* src/linker.cpp:209-258. Segments are visited in order and emit ascending indices,
 * so the reference's final std::sort is the identity here. */
uint32_t mo_select(uint32_t nseg, const uint8_t* kinds, const uint32_t* lens, int policy,
                   uint32_t k, int global, uint32_t* out) {
    uint32_t total = 0, m = 0, at = 0;
    for (uint32_t s = 0; s < nseg; ++s) total += lens[s];
    if (policy == 2) {
        for (uint32_t i = 0; i < total; ++i) out[i] = i;
        return total;
    }
    if (policy == 3) return 0;
    uint32_t budget = (policy == 0 && global) ? k : 0;
    for (uint32_t s = 0; s < nseg; ++s) {
        if (kinds[s] == 0) {
            for (uint32_t i = 0; i < lens[s]; ++i) out[m++] = at + i;
        } else if (policy == 0) {
            uint32_t take;
            if (global) {
                take = budget < lens[s] ? budget : lens[s];
                budget -= take;
            } else {
                take = k < lens[s] ? k : lens[s];
            }
            for (uint32_t i = 0; i < take; ++i) out[m++] = at + i;
        }
        at += lens[s];
    }
    return m;
}

/* src/model.cpp:46-62 (apply_rope) and :64-83 (rerotate_key): interleaved pairs,
 * angle in double, c/s rounded to float, products and sums in float. */
static void rotate_row(float* row, uint32_t heads, uint32_t dim, double delta, float base) {
    for (uint32_t hh = 0; hh < heads; ++hh) {
        float* hr = row + (size_t)hh * dim;
        for (uint32_t i = 0; i + 1 < dim; i += 2) {
            const double freq = pow((double)base, -(double)i / dim);
            const double theta = delta * freq;
            const float c = (float)cos(theta);
            const float s = (float)sin(theta);
            const float x0 = hr[i], x1 = hr[i + 1];
            hr[i] = x0 * c - x1 * s;
            hr[i + 1] = x0 * s + x1 * c;
        }
    }
}

/* src/linker.cpp:260-314 */
void mo_assemble(const mo_config* c, uint32_t nseg, const uint8_t* kinds, const uint32_t* lens,
                 const float* const* chunk_k, const float* const* chunk_v,
                 const uint32_t* chunk_base, int rerotate, float* out_k, float* out_v) {
    uint32_t n = 0;
    for (uint32_t s = 0; s < nseg; ++s) n += lens[s];
    const size_t row = (size_t)c->n_heads * c->head_dim;
    memset(out_k, 0, (size_t)c->n_layers * n * row * sizeof(float));
    memset(out_v, 0, (size_t)c->n_layers * n * row * sizeof(float));
    uint32_t at = 0, img = 0;
    for (uint32_t s = 0; s < nseg; ++s) {
        if (kinds[s] == 1) {
            const uint32_t len = lens[s];
            for (uint32_t l = 0; l < c->n_layers; ++l) {
                for (uint32_t j = 0; j < len; ++j) {
                    float* kd = out_k + ((size_t)l * n + at + j) * row;
                    memcpy(kd, chunk_k[img] + ((size_t)l * len + j) * row, row * sizeof(float));
                    const uint32_t from = chunk_base[img] + j, to = at + j;
                    if (rerotate && from != to)
                        rotate_row(kd, c->n_heads, c->head_dim, (double)to - (double)from,
                                   c->rope_base);
                    memcpy(out_v + ((size_t)l * n + at + j) * row,
                           chunk_v[img] + ((size_t)l * len + j) * row, row * sizeof(float));
                }
            }
            ++img;
        }
        at += lens[s];
    }
}

/* y[r] = sum_c W[r][c] x[c] for each of cnt rows: gemm_nt (src/matmul.cpp:7-13). */
static void gemm_nt(const float* x, uint32_t cnt, uint32_t in, const float* w, uint32_t out,
                    float* y) {
    for (uint32_t i = 0; i < cnt; ++i)
        for (uint32_t r = 0; r < out; ++r) {
            double acc = 0.0;
            const float* wr = w + (size_t)r * in;
            const float* xr = x + (size_t)i * in;
            for (uint32_t c = 0; c < in; ++c) acc += (double)wr[c] * xr[c];
            y[(size_t)i * out + r] = (float)acc;
        }
}

static float gelu(float x) { /* src/model.cpp:85-87 */
    return 0.5f * x * (1.0f + tanhf(0.7978845608028654f * (x + 0.044715f * x * x * x)));
}

/* src/linker.cpp:35-135 (selective_core); with rows = start+i and rope_pos =
 * base+start+i it is also src/model.cpp:211-330 (extend_rows). */
int mo_selective_core(const mo_model* m, const int32_t* ids, const uint32_t* rows,
                      const uint32_t* rope_pos, uint32_t cnt, float* kv_k, float* kv_v,
                      uint32_t n_ctx, float* logits) {
    const mo_config* c = &m->cfg;
    const uint32_t h = c->hidden_dim, heads = c->n_heads, dim = c->head_dim;
    const size_t row = h;
    if (cnt == 0) return -1;
    for (uint32_t i = 0; i < cnt; ++i)
        if (ids[i] < 0 || (uint32_t)ids[i] >= c->vocab_size) return -2; /* model.cpp:93-95 */
    float* x = (float*)malloc((size_t)cnt * h * sizeof(float));
    float* q = (float*)malloc((size_t)cnt * h * sizeof(float));
    float* t = (float*)malloc((size_t)cnt * h * sizeof(float));
    float* attn = (float*)malloc((size_t)cnt * h * sizeof(float));
    float* ffn = (float*)malloc((size_t)cnt * 4 * h * sizeof(float));
    float* s = (float*)malloc((size_t)(rows[cnt - 1] + 1) * sizeof(float));
    for (uint32_t i = 0; i < cnt; ++i)
        memcpy(x + (size_t)i * h, m->embedding + (size_t)ids[i] * h, h * sizeof(float));
    const float inv_sqrt_d = 1.0f / sqrtf((float)dim);

    for (uint32_t l = 0; l < c->n_layers; ++l) {
        float* const* w = m->w + 6 * l;
        float* kl = kv_k + (size_t)l * n_ctx * row;
        float* vl = kv_v + (size_t)l * n_ctx * row;
        gemm_nt(x, cnt, h, w[0], h, q);
        gemm_nt(x, cnt, h, w[1], h, t);
        for (uint32_t i = 0; i < cnt; ++i) {
            if (rope_pos[i] != 0) { /* rotation by angle 0 is the identity */
                rotate_row(q + (size_t)i * h, heads, dim, (double)rope_pos[i], c->rope_base);
                rotate_row(t + (size_t)i * h, heads, dim, (double)rope_pos[i], c->rope_base);
            }
            memcpy(kl + (size_t)rows[i] * row, t + (size_t)i * h, row * sizeof(float));
        }
        gemm_nt(x, cnt, h, w[2], h, t);
        for (uint32_t i = 0; i < cnt; ++i)
            memcpy(vl + (size_t)rows[i] * row, t + (size_t)i * h, row * sizeof(float));

        /* linker.cpp:80-113: every recomputed row is scattered before any attention. */
        for (uint32_t i = 0; i < cnt; ++i) {
            const uint32_t count = rows[i] + 1;
            for (uint32_t hh = 0; hh < heads; ++hh) {
                const float* qi = q + (size_t)i * h + (size_t)hh * dim;
                float mx = -INFINITY;
                for (uint32_t j = 0; j < count; ++j) {
                    const float* kj = kl + (size_t)j * row + (size_t)hh * dim;
                    double acc = 0.0;
                    for (uint32_t d = 0; d < dim; ++d) acc += (double)qi[d] * kj[d];
                    s[j] = (float)acc * inv_sqrt_d;
                    if (s[j] > mx) mx = s[j];
                }
                float sum = 0.0f;
                for (uint32_t j = 0; j < count; ++j) {
                    s[j] = expf(s[j] - mx);
                    sum += s[j];
                }
                for (uint32_t j = 0; j < count; ++j) s[j] /= sum;
                float* o = attn + (size_t)i * h + (size_t)hh * dim;
                for (uint32_t d = 0; d < dim; ++d) {
                    double acc = 0.0;
                    for (uint32_t j = 0; j < count; ++j)
                        acc += (double)s[j] * vl[(size_t)j * row + (size_t)hh * dim + d];
                    o[d] = (float)acc;
                }
            }
        }
        /* linker.cpp:115-128 */
        gemm_nt(attn, cnt, h, w[3], h, t);
        for (size_t e = 0; e < (size_t)cnt * h; ++e) x[e] += t[e];
        gemm_nt(x, cnt, h, w[4], 4 * h, ffn);
        for (size_t e = 0; e < (size_t)cnt * 4 * h; ++e) ffn[e] = gelu(ffn[e]);
        gemm_nt(ffn, cnt, 4 * h, w[5], h, t);
        for (size_t e = 0; e < (size_t)cnt * h; ++e) x[e] += t[e];
    }
    /* linker.cpp:131-133 */
    gemm_nt(x + (size_t)(cnt - 1) * h, 1, h, m->lm_head, c->vocab_size, logits);
    free(x); free(q); free(t); free(attn); free(ffn); free(s);
    return 0;
}
