// Diagnostic: the reference's "monotone work" scenario (proj/tests/test_linker.cpp:483-529)
// against libmpic_b200, printing every repetition's wall_ms per mask.
#include "mpic/linker.h"
#include "mpic/model.h"
#include "test_util.h"
#include <algorithm>
#include <cstdio>
#include <random>
using namespace mpic;
int main() {
    ModelConfig cfg;
    cfg.n_layers = 2; cfg.n_heads = 4; cfg.head_dim = 32; cfg.hidden_dim = 128;
    cfg.vocab_size = 512; cfg.image_token_count = 64; cfg.seed = 3;
    const Model model = build_model(cfg);
    std::mt19937_64 rng(10);
    SegmentedPrompt p;
    p.user = "u";
    std::vector<KvCacheEntry> entries;
    p.segments.push_back(Segment::text(testutil::random_ids(rng, 32, cfg.vocab_size)));
    for (int i = 0; i < 4; ++i) {
        KvCacheEntry e = testutil::make_image_entry(model, testutil::random_hash(rng), "u", 64, 0);
        p.segments.push_back(Segment::image(e.key, 64));
        entries.push_back(std::move(e));
    }
    p.segments.push_back(Segment::text(testutil::random_ids(rng, 32, cfg.vocab_size)));
    auto run = [&](const char* name, const SelectionMask& mask) {
        std::vector<double> t;
        for (int rep = 0; rep < 11; ++rep) {
            LinkedCache lc = assemble_linked_cache(p, entries, model);
            t.push_back(selective_prefill(model, p, mask, lc).stats.wall_ms);
        }
        std::printf("%s m=%zu:", name, mask.selected.size());
        for (double x : t) std::printf(" %.3f", x);
        std::sort(t.begin(), t.end());
        std::printf("  median %.3f\n", t[5]);
    };
    for (int round = 0; round < 2; ++round) {
        run("k0  ", select_tokens(p, MpicKPolicy{0}));
        run("k16 ", select_tokens(p, MpicKPolicy{16}));
        run("all ", select_tokens(p, AllPolicy{}));
    }
}
