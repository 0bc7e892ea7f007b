// Internal glue between the value-semantic mpic:: API and the C ABI: status -> exception
// mapping and RAII handles for device models, KV tensors and workspaces.
#pragma once

#include "mpic/errors.h"
#include "mpic/model.h"
#include "mpic/tensor.h"
#include "mpic_b200.h"

#include <string>

namespace mpic::b200 {

// Throws the mpic:: exception class matching an mpic_status (errors.h <-> mpic_b200.h).
void check(int rc);
int device();  // MPIC_DEVICE environment variable, default 0

mpic_model_config to_c(const ModelConfig& c);

class DeviceModel {
public:
    explicit DeviceModel(const Model& m);  // uploads the current host weights (fp32)
    ~DeviceModel();
    DeviceModel(const DeviceModel&) = delete;
    DeviceModel& operator=(const DeviceModel&) = delete;
    mpic_model_t get() const { return h_; }

private:
    mpic_model_t h_ = nullptr;
};

class DeviceKv {
public:
    DeviceKv(uint32_t layers, uint32_t tokens, uint32_t heads, uint32_t dim);
    explicit DeviceKv(const KvTensor& t);  // allocate + upload
    ~DeviceKv();
    DeviceKv(const DeviceKv&) = delete;
    DeviceKv& operator=(const DeviceKv&) = delete;
    void upload(const KvTensor& t);
    void download(KvTensor& t) const;  // t must have the matching shape
    mpic_kv_t get() const { return h_; }

private:
    mpic_kv_t h_ = nullptr;
};

class Workspace {
public:
    Workspace(const DeviceModel& m, uint32_t rows, uint32_t ctx);
    ~Workspace();
    Workspace(const Workspace&) = delete;
    Workspace& operator=(const Workspace&) = delete;
    mpic_workspace_t get() const { return h_; }

private:
    mpic_workspace_t h_ = nullptr;
};

}  // namespace mpic::b200
