// Diagnostic: the reference's "monotone work" scenario (proj/tests/test_linker.cpp:483-529)
// against libmpic_b200, printing every repetition's wall_ms per mask.
#include "mpic/linker.h"
#include "mpic/model.h"
#include "test_util.h"
#include "device.h"
#include <algorithm>
#include <chrono>
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
    // breakdown of one selective_prefill call (the steps of linker.cpp recompute_rows)
    {
        using clk = std::chrono::steady_clock;
        auto ms = [](clk::time_point a, clk::time_point b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
        const SelectionMask mask = select_tokens(p, MpicKPolicy{16});
        for (int rep = 0; rep < 5; ++rep) {
            LinkedCache lc = assemble_linked_cache(p, entries, model);
            const TokenIds flat = p.flatten_ids(model.config);
            const uint32_t m = mask.selected.size();
            TokenIds ids(m);
            for (uint32_t i = 0; i < m; ++i) ids[i] = flat[mask.selected[i]];
            auto t0 = clk::now();
            auto dm = b200::device_model_for(model);
            auto t1 = clk::now();
            b200::Workspace& ws = b200::workspace_for(dm, m, lc.kv.n_tokens);
            auto t2 = clk::now();
            auto* dkv = new b200::DeviceKv(lc.kv);
            auto t3 = clk::now();
            Logits logits(model.config.vocab_size);
            b200::check(mpic_selective_prefill(dm->get(), ws.get(), ids.data(), mask.selected.data(), m, dkv->get(), logits.data(), nullptr));
            auto t4 = clk::now();
            dkv->download(lc.kv);
            auto t5 = clk::now();
            delete dkv;
            auto t6 = clk::now();
            std::printf("model %.3f ws %.3f kv_alloc+up %.3f prefill %.3f down %.3f free %.3f\n", ms(t0, t1), ms(t1, t2), ms(t2, t3), ms(t3, t4), ms(t4, t5), ms(t5, t6));
        }
    }
    for (int round = 0; round < 2; ++round) {
        run("k0  ", select_tokens(p, MpicKPolicy{0}));
        run("k16 ", select_tokens(p, MpicKPolicy{16}));
        run("all ", select_tokens(p, AllPolicy{}));
    }
}
