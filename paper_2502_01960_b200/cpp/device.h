// Internal glue between the value-semantic mpic:: API and the C ABI: status -> exception
// mapping and RAII handles for device models, KV tensors and workspaces.
#pragma once

#include "mpic/errors.h"
#include "mpic/model.h"
#include "mpic/tensor.h"
#include "mpic_b200.h"

#include <memory>
#include <span>
#include <string>

namespace mpic::b200 {

// Throws the mpic:: exception class matching an mpic_status (errors.h <-> mpic_b200.h).
void check(int rc);
int device();  // MPIC_DEVICE environment variable, default 0
// Arithmetic of the drop-in API's device copies: fp32 (default: the reference's precision,
// SIMT kernels, the reference's own tests pass at their 1e-5 bars) or, with
// MPIC_B200_DTYPE=bf16, bf16 weights and KV — the tcgen05 GEMMs and (head_dim 128) the tcgen05
// attention, within the bf16 bar (1e-2). Host data stay fp32 either way.
mpic_dtype compute_dtype();

mpic_model_config to_c(const ModelConfig& c);

class DeviceModel {
public:
    explicit DeviceModel(const Model& m);  // uploads the current host weights (compute_dtype())
    ~DeviceModel();
    DeviceModel(const DeviceModel&) = delete;
    DeviceModel& operator=(const DeviceModel&) = delete;
    mpic_model_t get() const { return h_; }

private:
    mpic_model_t h_ = nullptr;
};

// Device KV tensors are recycled through a small per-thread pool keyed by shape, so the
// value-semantic API does not pay a cudaMalloc/cudaFree pair per call.
class DeviceKv {
public:
    DeviceKv(uint32_t layers, uint32_t tokens, uint32_t heads, uint32_t dim);
    explicit DeviceKv(const KvTensor& t);  // allocate + upload
    ~DeviceKv();
    DeviceKv(const DeviceKv&) = delete;
    DeviceKv& operator=(const DeviceKv&) = delete;
    void upload(const KvTensor& t);
    void download(KvTensor& t) const;  // t must have the matching shape
    // Only rows[] of every layer (the rows a selective pass rewrote).
    void download_rows(KvTensor& t, std::span<const uint32_t> rows) const;
    mpic_kv_t get() const { return h_; }

private:
    mpic_kv_t h_ = nullptr;
};

// Device copy of a host Model, cached across calls. The value-semantic API lets callers
// edit weights between calls (proj/tests/test_model.cpp zero_weights), so the cache key is
// the model's address, its config fingerprint and a 64-bit weight hash recomputed on each
// lookup; a mismatch re-uploads. The hash covers every weight word for models up to 64 Mi
// words (256 MB fp32: every test/conformance model); above that it samples each tensor
// (core.cpp weight_hash), so very large models must not be edited in place between calls.
std::shared_ptr<DeviceModel> device_model_for(const Model& m);

class Workspace {
public:
    Workspace(const DeviceModel& m, uint32_t rows, uint32_t ctx);
    ~Workspace();
    Workspace(const Workspace&) = delete;
    Workspace& operator=(const Workspace&) = delete;
    mpic_workspace_t get() const { return h_; }
    uint32_t rows() const { return rows_; }
    uint32_t ctx() const { return ctx_; }

private:
    mpic_workspace_t h_ = nullptr;
    uint32_t rows_ = 0, ctx_ = 0;
};

// Per-thread workspace reuse for a cached device model (grows on demand).
Workspace& workspace_for(const std::shared_ptr<DeviceModel>& m, uint32_t rows, uint32_t ctx);

}  // namespace mpic::b200
