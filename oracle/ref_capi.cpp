// Checker-side C ABI over the UNMODIFIED reference library (built from
// /root/reference/proj/src by oracle/Makefile). Test infrastructure only: tests/,
// __graft_entry__.smoke() and bench.py's reference arm load it through ctypes to
// run the reference's own functions on the same inputs as the B200 path.
// Every entry point forwards to the reference API named in its comment.
#include "mpic/cache.h"
#include "mpic/config.h"
#include "mpic/errors.h"
#include "mpic/linker.h"
#include "mpic/matmul.h"
#include "mpic/model.h"

#include <chrono>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

using namespace mpic;

namespace {
thread_local std::string g_err;

int fail(const std::exception& e) {
    g_err = e.what();
    if (dynamic_cast<const config_error*>(&e)) return 1;
    if (dynamic_cast<const validation_error*>(&e)) return 2;
    if (dynamic_cast<const state_error*>(&e)) return 3;
    if (dynamic_cast<const link_error*>(&e)) return 4;
    if (dynamic_cast<const contract_error*>(&e)) return 5;
    if (dynamic_cast<const format_error*>(&e)) return 6;
    if (dynamic_cast<const integrity_error*>(&e)) return 7;
    if (dynamic_cast<const io_error*>(&e)) return 8;
    if (dynamic_cast<const not_found_error*>(&e)) return 9;
    return 99;
}

ModelConfig make_cfg(const uint32_t* u, float rope_base, uint64_t seed) {
    ModelConfig c;
    c.n_layers = u[0];
    c.n_heads = u[1];
    c.head_dim = u[2];
    c.hidden_dim = u[3];
    c.vocab_size = u[4];
    c.image_token_count = u[5];
    c.rope_base = rope_base;
    c.seed = seed;
    return c;
}

// Prompt descriptor: nseg segments; kinds[i] 0=text 1=image; lens[i] tokens;
// text ids concatenated in segment order; 32-byte content hashes per image.
SegmentedPrompt make_prompt(const Model& m, uint32_t nseg, const uint8_t* kinds,
                            const uint32_t* lens, const int32_t* text_ids,
                            const uint8_t* hashes, const char* ns) {
    SegmentedPrompt p;
    p.user = ns ? ns : "";
    size_t ti = 0, hi = 0;
    for (uint32_t s = 0; s < nseg; ++s) {
        if (kinds[s] == 0) {
            p.segments.push_back(Segment::text(TokenIds(text_ids + ti, text_ids + ti + lens[s])));
            ti += lens[s];
        } else {
            CacheKey key;
            std::memcpy(key.content_hash.data(), hashes + 32 * hi, 32);
            key.model_fingerprint = m.config.fingerprint();
            key.ns = p.user;
            ++hi;
            p.segments.push_back(Segment::image(key, lens[s]));
        }
    }
    return p;
}

struct Entries {
    std::vector<KvCacheEntry> v;
};
} // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// mpic::set_compute_threads (proj/include/mpic/matmul.h:23)
void ref_set_threads(int n) { set_compute_threads(n); }

// ModelConfig::fingerprint (proj/src/config.cpp:30-47)
uint64_t ref_fingerprint(const uint32_t* u6, float rope_base, uint64_t seed) {
    return make_cfg(u6, rope_base, seed).fingerprint();
}

// build_model (proj/src/model.cpp:103-123)
int ref_model_create(const uint32_t* u6, float rope_base, uint64_t seed, void** out) {
    try {
        *out = new Model(build_model(make_cfg(u6, rope_base, seed)));
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}
void ref_model_free(void* m) { delete static_cast<Model*>(m); }

// Pointer to a weight matrix; which: 0 emb,1 lm_head,2 wq,3 wk,4 wv,5 wo,6 w1,7 w2.
const float* ref_model_weight(void* h, int which, uint32_t layer) {
    Model& m = *static_cast<Model*>(h);
    switch (which) {
        case 0: return m.embedding.data();
        case 1: return m.lm_head.data();
        case 2: return m.layers[layer].wq.data();
        case 3: return m.layers[layer].wk.data();
        case 4: return m.layers[layer].wv.data();
        case 5: return m.layers[layer].wo.data();
        case 6: return m.layers[layer].w1.data();
        case 7: return m.layers[layer].w2.data();
    }
    return nullptr;
}
uint64_t ref_weight_checksum(void* h) { return static_cast<Model*>(h)->weight_checksum(); }

// image_token_ids (proj/src/model.cpp:148-156)
void ref_image_ids(void* h, const uint8_t* hash32, uint32_t count, int32_t* out) {
    Hash256 hh;
    std::memcpy(hh.data(), hash32, 32);
    TokenIds ids = image_token_ids(hh, static_cast<Model*>(h)->config, count);
    std::memcpy(out, ids.data(), count * sizeof(int32_t));
}

// prefill_extend on an empty cache (proj/src/model.cpp:334-349): the standalone
// chunk precompute. k/v out: [L][n][H*D]; logits out: [V].
int ref_prefill(void* h, const int32_t* ids, uint32_t n, uint32_t base, float* k, float* v,
                float* logits) {
    try {
        const Model& m = *static_cast<Model*>(h);
        PrefillResult r = prefill_extend(m, std::span<const int32_t>(ids, n), KvTensor(), base);
        std::memcpy(k, r.kv.k.data(), r.kv.k.size() * sizeof(float));
        std::memcpy(v, r.kv.v.data(), r.kv.v.size() * sizeof(float));
        std::memcpy(logits, r.logits.data(), r.logits.size() * sizeof(float));
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// Chunk entries (KvCacheEntry, proj/include/mpic/cache.h:38-49) in input order.
void* ref_entries_create() { return new Entries(); }
void ref_entries_free(void* e) { delete static_cast<Entries*>(e); }
int ref_entries_add(void* eh, void* h, const uint8_t* hash32, const char* ns, uint32_t tokens,
                    uint32_t position_base, const float* k, const float* v) {
    const Model& m = *static_cast<Model*>(h);
    KvCacheEntry e;
    std::memcpy(e.key.content_hash.data(), hash32, 32);
    e.key.model_fingerprint = m.config.fingerprint();
    e.key.ns = ns ? ns : "";
    e.kv = KvTensor(m.config.n_layers, tokens, m.config.n_heads, m.config.head_dim);
    std::memcpy(e.kv.k.data(), k, e.kv.k.size() * sizeof(float));
    std::memcpy(e.kv.v.data(), v, e.kv.v.size() * sizeof(float));
    e.token_count = tokens;
    e.position_base = position_base;
    static_cast<Entries*>(eh)->v.push_back(std::move(e));
    return 0;
}

// select_tokens (proj/src/linker.cpp:209-258). policy: 0 MpicK, 1 TextOnly, 2 All,
// 3 PrefixOnly. out needs total_tokens slots; *m_out gets |mask|.
int ref_select(void* h, uint32_t nseg, const uint8_t* kinds, const uint32_t* lens,
               const int32_t* text_ids, const uint8_t* hashes, int policy, uint32_t k,
               int global, uint32_t* out, uint32_t* m_out) {
    try {
        const Model& m = *static_cast<Model*>(h);
        SegmentedPrompt p = make_prompt(m, nseg, kinds, lens, text_ids, hashes, "");
        SelectionPolicy pol;
        if (policy == 0) pol = MpicKPolicy{k, global != 0};
        else if (policy == 1) pol = TextOnlyPolicy{};
        else if (policy == 2) pol = AllPolicy{};
        else pol = PrefixOnlyPolicy{};
        SelectionMask mask = select_tokens(p, pol);
        std::memcpy(out, mask.selected.data(), mask.selected.size() * sizeof(uint32_t));
        *m_out = static_cast<uint32_t>(mask.selected.size());
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// flatten_ids (proj/src/linker.cpp:160-172)
int ref_flatten(void* h, uint32_t nseg, const uint8_t* kinds, const uint32_t* lens,
                const int32_t* text_ids, const uint8_t* hashes, int32_t* out) {
    try {
        const Model& m = *static_cast<Model*>(h);
        SegmentedPrompt p = make_prompt(m, nseg, kinds, lens, text_ids, hashes, "");
        TokenIds ids = p.flatten_ids(m.config);
        std::memcpy(out, ids.data(), ids.size() * sizeof(int32_t));
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// assemble_linked_cache (proj/src/linker.cpp:260-314) followed, when mask != NULL, by
// selective_prefill (proj/src/linker.cpp:316-353). Outputs: assembled KV (before the
// selective pass) into asm_k/asm_v if non-null; final KV into fin_k/fin_v if non-null;
// slots as (kind, entry_index, local_index) triples; logits [V]. Wall times of the two
// reference calls in ms go to ms_out[0..1].
int ref_link_and_prefill(void* h, uint32_t nseg, const uint8_t* kinds, const uint32_t* lens,
                         const int32_t* text_ids, const uint8_t* hashes, const char* ns,
                         void* entries, int rerotate, const uint32_t* mask, uint32_t m,
                         float* asm_k, float* asm_v, float* fin_k, float* fin_v,
                         uint32_t* slots, float* logits, double* ms_out) {
    try {
        const Model& mdl = *static_cast<Model*>(h);
        SegmentedPrompt p = make_prompt(mdl, nseg, kinds, lens, text_ids, hashes, ns);
        const auto& ents = static_cast<Entries*>(entries)->v;
        LinkOptions opt;
        opt.reposition = rerotate ? Reposition::Rerotate : Reposition::AsStored;
        const auto t0 = std::chrono::steady_clock::now();
        LinkedCache lc = assemble_linked_cache(p, ents, mdl, opt);
        const auto t1 = std::chrono::steady_clock::now();
        if (ms_out) ms_out[0] = std::chrono::duration<double, std::milli>(t1 - t0).count();
        if (asm_k) std::memcpy(asm_k, lc.kv.k.data(), lc.kv.k.size() * sizeof(float));
        if (asm_v) std::memcpy(asm_v, lc.kv.v.data(), lc.kv.v.size() * sizeof(float));
        if (mask) {
            SelectionMask sm;
            sm.selected.assign(mask, mask + m);
            const auto t2 = std::chrono::steady_clock::now();
            SelectiveResult r = selective_prefill(mdl, p, sm, lc);
            const auto t3 = std::chrono::steady_clock::now();
            if (ms_out) ms_out[1] = std::chrono::duration<double, std::milli>(t3 - t2).count();
            if (logits) std::memcpy(logits, r.logits.data(), r.logits.size() * sizeof(float));
        }
        if (fin_k) std::memcpy(fin_k, lc.kv.k.data(), lc.kv.k.size() * sizeof(float));
        if (fin_v) std::memcpy(fin_v, lc.kv.v.data(), lc.kv.v.size() * sizeof(float));
        if (slots) {
            for (size_t i = 0; i < lc.slots.size(); ++i) {
                slots[3 * i] = static_cast<uint32_t>(lc.slots[i].kind);
                slots[3 * i + 1] = lc.slots[i].entry_index;
                slots[3 * i + 2] = lc.slots[i].local_index;
            }
        }
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// serialize_entry (proj/src/cache.cpp:97-124) of entry #idx: returns the byte count;
// writes when out != NULL.
uint64_t ref_serialize_entry(void* entries, uint32_t idx, uint8_t* out) {
    std::vector<uint8_t> b = serialize_entry(static_cast<Entries*>(entries)->v.at(idx));
    if (out) std::memcpy(out, b.data(), b.size());
    return b.size();
}

} // extern "C"
