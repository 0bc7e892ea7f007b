// The reference's own API (include/mpic) end to end — MPIC-k selective prefill, CacheBlend
// selection + its selective prefill, full reuse, decode — printing every result as text so
// tests/test_gpu_cpp.py can run it twice (MPIC_B200_DTYPE unset: fp32 SIMT path; =bf16:
// tcgen05 GEMMs + tcgen05 attention, head_dim 128) and compare the two within the bf16 bar.
// Shape: L2 H4 D128 V2048, two 200-token images interleaved with text.
#include "mpic/linker.h"
#include "mpic/model.h"

#include <cstdio>
#include <vector>

static void dump(const char* tag, const std::vector<float>& v) {
    std::printf("%s %zu", tag, v.size());
    for (float x : v) std::printf(" %.9g", x);
    std::printf("\n");
}

int main() {
    mpic::ModelConfig cfg;
    cfg.n_layers = 2;
    cfg.n_heads = 4;
    cfg.head_dim = 128;
    cfg.hidden_dim = 512;
    cfg.vocab_size = 2048;
    cfg.image_token_count = 200;
    cfg.seed = 21;
    const mpic::Model model = mpic::build_model(cfg);
    std::vector<mpic::KvCacheEntry> entries;
    mpic::SegmentedPrompt prompt;
    prompt.segments.push_back(mpic::Segment::text({5, 17, 99, 3, 1000, 42, 7, 8, 9, 10, 11, 12}));
    for (int i = 0; i < 2; ++i) {
        mpic::CacheKey key;
        for (int b = 0; b < 32; ++b) key.content_hash[b] = static_cast<uint8_t>(31 * i + 7 * b + 1);
        key.model_fingerprint = cfg.fingerprint();
        key.ns = "dynamic";
        const mpic::TokenIds ids = mpic::image_token_ids(key.content_hash, cfg);
        mpic::KvCacheEntry e;
        e.key = key;
        e.token_count = cfg.image_token_count;
        e.kv = mpic::prefill_extend(model, ids, mpic::KvTensor{}).kv;  // precomputed at base 0
        entries.push_back(std::move(e));
        prompt.segments.push_back(mpic::Segment::image(key, cfg.image_token_count));
        prompt.segments.push_back(mpic::Segment::text({int32_t(100 + i), int32_t(200 + i), 300, 400, 500}));
    }
    // MPIC-k (the paper's policy) through assemble_linked_cache + selective_prefill
    const mpic::SelectionMask mk = mpic::select_tokens(prompt, mpic::MpicKPolicy{16});
    mpic::LinkedCache linked = mpic::assemble_linked_cache(prompt, entries, model);
    const auto r1 = mpic::selective_prefill(model, prompt, mk, linked);
    dump("mpick_logits", r1.logits);
    // CacheBlend-r (its selection is data-dependent: print it; compare only when equal)
    const mpic::SelectionMask cb = mpic::cacheblend_select(model, prompt, entries, 15.0);
    std::printf("cacheblend_sel %zu", cb.selected.size());
    for (uint32_t s : cb.selected) std::printf(" %u", s);
    std::printf("\n");
    mpic::LinkedCache linked2 = mpic::assemble_linked_cache(prompt, entries, model);
    const auto r2 = mpic::selective_prefill(model, prompt, cb, linked2);
    dump("cacheblend_logits", r2.logits);
    // full reuse (no recomputation beyond the final token's requirement)
    const auto fr = mpic::full_reuse_prefill(model, prompt, entries);
    dump("full_reuse_logits", fr.logits);
    // decode two tokens after the MPIC-k prefill
    mpic::KvTensor cache = std::move(linked.kv);
    const uint32_t n = prompt.total_tokens();
    const auto d1 = mpic::decode_step(model, cache, 77, n);
    const auto d2 = mpic::decode_step(model, cache, 1234, n + 1);
    dump("decode1_logits", d1);
    dump("decode2_logits", d2);
    return 0;
}
