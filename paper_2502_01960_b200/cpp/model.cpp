// mpic:: model API on the B200 path (proj/include/mpic/model.h semantics).
#include "device.h"

#include "mpic/errors.h"
#include "mpic/model.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <string>

namespace mpic {

namespace {

// One forward over rows [start, start+m) of a cache of n = start+m rows (extend_rows,
// proj/src/model.cpp:211-330): positions base+start+i. Optional hidden rows / capture.
PrefillResult extend(const Model& model, std::span<const int32_t> ids, KvTensor&& cache,
                     uint32_t position_base, AttentionDump* capture, std::vector<float>* hidden) {
    const ModelConfig& c = model.config;
    const uint32_t m = static_cast<uint32_t>(ids.size());
    if (m == 0) throw validation_error("no tokens to prefill");
    for (const int32_t id : ids)
        if (id < 0 || static_cast<uint32_t>(id) >= c.vocab_size)
            throw validation_error("token id " + std::to_string(id) + " out of vocabulary");
    if (cache.n_tokens == 0) {
        cache = KvTensor(c.n_layers, 0, c.n_heads, c.head_dim);
    } else if (cache.n_layers != c.n_layers || cache.n_heads != c.n_heads || cache.head_dim != c.head_dim) {
        throw validation_error("cache shape does not match model");
    }
    const uint32_t start = cache.n_tokens;
    PrefillResult res;
    res.kv = std::move(cache);
    res.kv.resize_tokens(start + m);
    const uint32_t n = start + m;

    const auto dm = b200::device_model_for(model);
    b200::Workspace& ws = b200::workspace_for(dm, m, n);
    b200::DeviceKv kv(res.kv);
    std::vector<uint32_t> rows(m), pos(m);
    for (uint32_t i = 0; i < m; ++i) {
        rows[i] = start + i;
        pos[i] = position_base + start + i;
    }
    res.logits.assign(c.vocab_size, 0.0f);
    if (hidden) hidden->assign(size_t(m) * c.hidden_dim, 0.0f);
    if (capture) {
        capture->n_layers = c.n_layers;
        capture->n_heads = c.n_heads;
        capture->n_tokens = n;
        capture->model_fingerprint = c.fingerprint();
        capture->scores.assign(size_t(c.n_layers) * c.n_heads * n * n, 0.0f);
    }
    b200::check(mpic_forward_rows(dm->get(), ws.get(), ids.data(), rows.data(), pos.data(), m, kv.get(),
                                  res.logits.data(), hidden ? hidden->data() : nullptr,
                                  capture ? capture->scores.data() : nullptr, nullptr));
    kv.download(res.kv);
    return res;
}

}  // namespace

// build_model (model.cpp:103-123): synthesised on the device, mirrored to host vectors.
Model build_model(const ModelConfig& config) {
    config.validate();
    const mpic_model_config c = b200::to_c(config);
    mpic_model_t h = nullptr;
    b200::check(mpic_model_create(&c, b200::device(), MPIC_F32, &h));
    Model m;
    m.config = config;
    const size_t hd = config.hidden_dim, V = config.vocab_size;
    try {
        m.embedding.resize(V * hd);
        m.lm_head.resize(V * hd);
        b200::check(mpic_model_download_weight(h, 0, 0, m.embedding.data()));
        b200::check(mpic_model_download_weight(h, 1, 0, m.lm_head.data()));
        m.layers.resize(config.n_layers);
        for (uint32_t l = 0; l < config.n_layers; ++l) {
            LayerWeights& w = m.layers[l];
            std::vector<float>* mats[6] = {&w.wq, &w.wk, &w.wv, &w.wo, &w.w1, &w.w2};
            for (int i = 0; i < 6; ++i) {
                mats[i]->resize(i >= 4 ? 4 * hd * hd : hd * hd);
                b200::check(mpic_model_download_weight(h, 2 + i, l, mats[i]->data()));
            }
        }
    } catch (...) {
        mpic_model_destroy(h);
        throw;
    }
    mpic_model_destroy(h);
    return m;
}

uint64_t Model::weight_checksum() const {
    uint64_t acc = 0xcbf29ce484222325ull;
    auto feed = [&](const std::vector<float>& w) {
        const auto* p = reinterpret_cast<const uint8_t*>(w.data());
        for (size_t i = 0, n = w.size() * sizeof(float); i < n; ++i) acc = (acc ^ p[i]) * 0x100000001b3ull;
    };
    feed(embedding);
    feed(lm_head);
    for (const LayerWeights& l : layers)
        for (const std::vector<float>* w : {&l.wq, &l.wk, &l.wv, &l.wo, &l.w1, &l.w2}) feed(*w);
    return acc;
}

TokenIds image_token_ids(const Hash256& content_hash, const ModelConfig& config, uint32_t count) {
    const mpic_model_config c = b200::to_c(config);
    TokenIds ids(count);
    b200::check(mpic_image_token_ids(&c, content_hash.data(), count, ids.data()));
    return ids;
}

TokenIds image_token_ids(const Hash256& content_hash, const ModelConfig& config) {
    return image_token_ids(content_hash, config, config.image_token_count);
}

TokenIds encode_image(std::span<const uint8_t> image_bytes, const ModelConfig& config) {
    if (image_bytes.empty()) throw validation_error("image bytes must be non-empty");
    return image_token_ids(sha256(image_bytes), config);
}

// Scalar helper (model.cpp:169-198): one softmax row, used by tests and diagnostics.
std::vector<float> attention_row(std::span<const float> q, std::span<const std::vector<float>> keys,
                                 uint32_t head_dim) {
    if (q.size() != head_dim) throw validation_error("query length does not match head_dim");
    const float scale = 1.0f / std::sqrt(static_cast<float>(head_dim));
    std::vector<float> p(keys.size());
    float top = -std::numeric_limits<float>::infinity();
    for (size_t j = 0; j < keys.size(); ++j) {
        if (keys[j].size() != head_dim) throw validation_error("key length does not match head_dim");
        float dot = 0.0f;
        for (uint32_t d = 0; d < head_dim; ++d) dot += q[d] * keys[j][d];
        p[j] = dot * scale;
        top = std::max(top, p[j]);
    }
    float total = 0.0f;
    for (float& x : p) total += (x = std::exp(x - top));
    for (float& x : p) x /= total;
    return p;
}

PrefillResult prefill_extend(const Model& model, std::span<const int32_t> ids, KvTensor&& cache,
                             uint32_t position_base, AttentionDump* capture) {
    return extend(model, ids, std::move(cache), position_base, capture, nullptr);
}

PrefillResult full_prefill(const Model& model, std::span<const int32_t> ids, AttentionDump* capture) {
    return prefill_extend(model, ids, KvTensor(), 0, capture);
}

Logits decode_step(const Model& model, KvTensor& cache, int32_t next_token, uint32_t position,
                   uint32_t position_base) {
    if (position != position_base + cache.n_tokens)
        throw state_error("decode position " + std::to_string(position) + " does not match cache length " +
                          std::to_string(position_base + cache.n_tokens));
    const int32_t one[1] = {next_token};
    PrefillResult r = prefill_extend(model, one, std::move(cache), position_base);
    cache = std::move(r.kv);
    return std::move(r.logits);
}

std::vector<float> mean_pooled_hidden(const Model& model, std::span<const int32_t> ids) {
    const uint32_t hd = model.config.hidden_dim;
    std::vector<float> pooled(hd, 0.0f);
    if (ids.empty()) return pooled;
    std::vector<float> rows;
    extend(model, ids, KvTensor(), 0, nullptr, &rows);
    for (size_t i = 0; i < ids.size(); ++i)
        for (uint32_t d = 0; d < hd; ++d) pooled[d] += rows[i * hd + d];
    for (float& x : pooled) x /= static_cast<float>(ids.size());
    return pooled;
}

int32_t argmax_token(std::span<const float> logits) {
    if (logits.empty()) return 0;
    return static_cast<int32_t>(std::max_element(logits.begin(), logits.end()) - logits.begin());
}

namespace detail {

// Host copies of the rotation/activation helpers (model.cpp:46-99) for callers that work
// on host rows; the device kernels implement the same arithmetic (common.cuh).
static void rotate(float* row, uint32_t heads, uint32_t dim, double delta, float base) {
    for (uint32_t hh = 0; hh < heads; ++hh) {
        float* r = row + size_t(hh) * dim;
        for (uint32_t i = 0; i + 1 < dim; i += 2) {
            const double theta = delta * std::pow(static_cast<double>(base), -static_cast<double>(i) / dim);
            const float c = static_cast<float>(std::cos(theta)), s = static_cast<float>(std::sin(theta));
            const float x0 = r[i], x1 = r[i + 1];
            r[i] = x0 * c - x1 * s;
            r[i + 1] = x0 * s + x1 * c;
        }
    }
}

void apply_rope(float* row, uint32_t n_heads, uint32_t head_dim, uint32_t position, float rope_base) {
    rotate(row, n_heads, head_dim, static_cast<double>(position), rope_base);
}

void rerotate_key(float* row, uint32_t n_heads, uint32_t head_dim, uint32_t from, uint32_t to,
                  float rope_base) {
    if (from == to) return;
    rotate(row, n_heads, head_dim, static_cast<double>(to) - static_cast<double>(from), rope_base);
}

float gelu(float x) {
    return 0.5f * x * (1.0f + std::tanh(0.7978845608028654f * (x + 0.044715f * x * x * x)));
}

void embed_tokens(const Model& model, std::span<const int32_t> ids, float* out) {
    const uint32_t hd = model.config.hidden_dim;
    for (size_t i = 0; i < ids.size(); ++i) {
        const int32_t id = ids[i];
        if (id < 0 || static_cast<uint32_t>(id) >= model.config.vocab_size)
            throw validation_error("token id " + std::to_string(id) + " out of vocabulary");
        std::memcpy(out + i * hd, model.embedding.data() + size_t(id) * hd, hd * sizeof(float));
    }
}

}  // namespace detail
}  // namespace mpic
