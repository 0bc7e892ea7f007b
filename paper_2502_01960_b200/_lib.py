"""ctypes binding of the C ABI in include/mpic_b200.h (libmpic_b200.so, built in-tree).

The library is required: importing works without it (so CPU-only tooling can inspect
the package), but every call raises ``ExtensionMissing`` when it was not built — there
is no CPU fallback anywhere on the product path.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_DIR = os.path.join(HERE, "lib")
LIB_PATH = os.environ.get("MPIC_B200_LIB") or os.path.join(LIB_DIR, "libmpic_b200.so")  # env: diagnostics builds


class ExtensionMissing(RuntimeError):
    pass


class MpicError(RuntimeError):
    """Raised for a non-zero mpic_status; ``code`` maps onto the reference's exception
    classes (proj/include/mpic/errors.h:10-62)."""

    NAMES = {1: "config_error", 2: "validation_error", 3: "state_error", 4: "link_error",
             5: "contract_error", 6: "format_error", 7: "integrity_error", 8: "io_error",
             9: "not_found_error", 10: "request_error", 20: "cuda_error", 21: "no_device"}

    def __init__(self, code: int, msg: str):
        super().__init__(f"{self.NAMES.get(code, code)}: {msg}")
        self.code = code
        self.kind = self.NAMES.get(code, str(code))


class ModelConfig(C.Structure):
    """mpic_model_config == mpic::ModelConfig (proj/include/mpic/config.h:7-24)."""

    _fields_ = [("n_layers", C.c_uint32), ("n_heads", C.c_uint32), ("head_dim", C.c_uint32),
                ("hidden_dim", C.c_uint32), ("vocab_size", C.c_uint32),
                ("image_token_count", C.c_uint32), ("rope_base", C.c_float), ("seed", C.c_uint64)]


class ChunkRef(C.Structure):
    _fields_ = [("src", C.c_void_p), ("src_row0", C.c_uint32), ("dst_row0", C.c_uint32),
                ("rows", C.c_uint32), ("position_base", C.c_uint32)]


class PromptDesc(C.Structure):
    _fields_ = [("n_segments", C.c_uint32), ("kinds", C.c_void_p), ("lens", C.c_void_p),
                ("text_ids", C.c_void_p), ("hashes", C.c_void_p)]


class PolicyDesc(C.Structure):
    _fields_ = [("policy", C.c_int), ("k", C.c_uint32), ("global_budget", C.c_int)]


_vp, _u32, _i32, _f, _int = C.c_void_p, C.c_uint32, C.c_int32, C.c_float, C.c_int
_P = C.POINTER

# name -> (restype, argtypes); mirrors include/mpic_b200.h
SIGNATURES = {
    "mpic_last_error": (C.c_char_p, []),
    "mpic_version": (C.c_char_p, []),
    "mpic_last_launch_count": (_u32, []),
    "mpic_config_validate": (_int, [_P(ModelConfig)]),
    "mpic_config_fingerprint": (C.c_uint64, [_P(ModelConfig)]),
    "mpic_model_create": (_int, [_P(ModelConfig), _int, _int, _P(_vp)]),
    "mpic_model_upload": (_int, [_P(ModelConfig), _int, _int, _vp, _vp, _vp, _P(_vp)]),
    "mpic_model_destroy": (_int, [_vp]),
    "mpic_model_config_get": (_int, [_vp, _P(ModelConfig)]),
    "mpic_model_dtype": (_int, [_vp]),
    "mpic_model_device": (_int, [_vp]),
    "mpic_store_create": (_int, [_vp, C.c_char_p, _u32, _u32, _P(_vp)]),
    "mpic_store_destroy": (_int, [_vp]),
    "mpic_store_put": (_int, [_vp, _vp, C.c_char_p, _vp, _u32]),
    "mpic_store_tier": (_int, [_vp, _vp, C.c_char_p, _P(_int)]),
    "mpic_store_demote": (_int, [_vp, _vp, C.c_char_p, _int]),
    "mpic_store_remove": (_int, [_vp, _vp, C.c_char_p]),
    "mpic_store_request": (_int, [_vp, _vp, _P(PromptDesc), _P(PolicyDesc), C.c_char_p, _int, _vp, _vp, _vp,
                                  _P(_u32), _vp, _vp]),
    "mpic_crc32_device": (_int, [_vp, C.c_size_t, _P(_u32), _vp]),
    "mpic_crc32_planes_device": (_int, [_vp, C.c_size_t, _u32, _vp, _vp]),
    "mpic_model_download_weight": (_int, [_vp, _int, _u32, _vp]),
    "mpic_kv_alloc": (_int, [_u32, _u32, _u32, _u32, _int, _int, _P(_vp)]),
    "mpic_kv_free": (_int, [_vp]),
    "mpic_kv_shape": (_int, [_vp, _vp, _P(_int)]),
    "mpic_kv_device_ptrs": (_int, [_vp, _P(_vp), _P(_vp)]),
    "mpic_kv_upload": (_int, [_vp, _vp, _vp, _vp]),
    "mpic_kv_download": (_int, [_vp, _vp, _vp, _vp]),
    "mpic_kv_zero_rows": (_int, [_vp, _u32, _u32, _vp]),
    "mpic_assemble": (_int, [_vp, _vp, _u32, _vp, _int, _f, _int]),
    "mpic_assemble_raw": (_int, [_vp, _vp, _vp, _vp, _int, _vp, _u32, _vp, _int, _f, _int]),
    "mpic_workspace_create": (_int, [_vp, _u32, _u32, _P(_vp)]),
    "mpic_workspace_destroy": (_int, [_vp]),
    "mpic_selective_prefill": (_int, [_vp, _vp, _vp, _vp, _u32, _vp, _vp, _vp]),
    "mpic_prefill_extend": (_int, [_vp, _vp, _vp, _u32, _u32, _u32, _vp, _vp, _vp]),
    "mpic_forward_rows": (_int, [_vp, _vp, _vp, _vp, _vp, _u32, _vp, _vp, _vp, _vp, _vp]),
    "mpic_layer0_keys": (_int, [_vp, _vp, _vp, _vp, _u32, _vp, _vp]),
    "mpic_forward_rows_async": (_int, [_vp, _vp, _vp, _vp, _vp, _u32, _u32, _vp, _vp, _vp]),
    "mpic_image_token_ids": (_int, [_P(ModelConfig), _vp, _u32, _vp]),
    "mpic_select_tokens": (_int, [_P(PromptDesc), _P(PolicyDesc), _vp, _P(_u32)]),
    "mpic_flatten_ids": (_int, [_P(ModelConfig), _P(PromptDesc), _vp]),
    "mpic_request_prefill": (_int, [_vp, _vp, _P(PromptDesc), _P(PolicyDesc), _vp, _int, _vp,
                                    _vp, _vp, _vp, _P(_u32), _vp]),
    "mpic_request_prefill_host": (_int, [_vp, _vp, _P(PromptDesc), _P(PolicyDesc), _vp, _vp,
                                         _vp, _int, _vp, _vp, _vp, _P(_u32), _vp]),
    "mpic_kv_download_rows": (_int, [_vp, _vp, _u32, _vp, _vp, _vp]),
    "mpic_workspace_set_graphs": (_int, [_vp, _int]),
    "mpic_request_prefill_batch": (_int, [_vp, _vp, _P(PromptDesc), _u32, _P(PolicyDesc), _vp, _int, _vp, _vp,
                                          _vp, _vp]),
    "mpic_request_prefill_files": (_int, [_vp, _vp, _P(PromptDesc), _P(PolicyDesc), _vp, _int, _vp, _vp, _vp,
                                          _P(_u32), _vp]),
    "mpic_request_prefill_files2": (_int, [_vp, _vp, _P(PromptDesc), _P(PolicyDesc), _vp, _int, _vp, _vp, _vp,
                                           _P(_u32), _vp, _vp]),
    "mpic_request_prefill_host2": (_int, [_vp, _vp, _P(PromptDesc), _P(PolicyDesc), _vp, _vp, _int, _vp,
                                          _int, _vp, _vp, _vp, _P(_u32), _vp]),
    "mpic_model_create_heads": (_int, [_P(ModelConfig), _int, _int, _u32, _u32, _P(_vp)]),
    "mpic_hp_prepare": (_int, [_vp, _vp, _P(PromptDesc), _P(PolicyDesc), _vp, _int, _vp, _vp, _vp, _P(_u32), _vp]),
    "mpic_hp_layer_attn": (_int, [_vp, _vp, _u32, _vp, _vp, _vp]),
    "mpic_hp_layer_ffn": (_int, [_vp, _vp, _u32, _vp, _u32, _u32, _vp]),
    "mpic_hp_logits": (_int, [_vp, _vp, _u32, _vp, _vp]),
    "mpic_workspace_device_ptr": (_int, [_vp, _int, _P(_vp)]),
    "mpic_hp_request": (_int, [_vp, _vp, _vp, _P(PromptDesc), _P(PolicyDesc), _vp, _int, _vp, _vp, _vp, _vp,
                               _P(_u32), _vp]),
    "mpic_nccl_unique_id": (_int, [_vp]),
    "mpic_nccl_comm_create": (_int, [_vp, _int, _int, _int, _P(_vp)]),
    "mpic_nccl_comm_destroy": (_int, [_vp]),
    "mpic_clock_probe": (_int, [_vp, _u32, _vp]),
    "mpic_pgemm_timestamps": (_int, [_vp]),
    "mpic_test_gemm": (_int, [_vp, _vp, _u32, _u32, _u32, _int, _vp, _vp]),
    "mpic_test_gemm_epi": (_int, [_vp, _vp, _u32, _u32, _u32, _int, _vp, _vp, _vp, _vp]),
    "mpic_test_qkv": (_int, [_vp, _vp, _u32, _u32, _u32, _u32, _vp, _vp, _vp, _vp, _vp, _vp]),
    "mpic_profile_enable": (_int, [_int]),
    "mpic_profile_collect": (_int, [_vp, _vp]),
    "mpic_test_attention": (_int, [_vp, _vp, _vp, _vp, _u32, _u32, _u32, _vp, _vp]),
    "mpic_attention_plan": (_int, [_vp, _u32, _u32, _vp, _vp, _vp, _u32, _vp, _u32, _vp, _u32]),
    "mpic_host_gemm_f32": (_int, [_vp, _vp, _u32, _u32, _u32, _vp, _int]),
    "mpic_host_alloc": (_int, [C.c_size_t, _P(_vp)]),
    "mpic_host_free": (_int, [_vp]),
}

_lib = None


def lib():
    """Load libmpic_b200.so (raises ExtensionMissing when it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ExtensionMissing(
                f"{LIB_PATH} not built — run __graft_entry__.build(); there is no CPU fallback")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(rc: int):
    if rc != 0:
        raise MpicError(rc, lib().mpic_last_error().decode(errors="replace"))
