"""ctypes binding of libtierkv_b200.so (include/tierkv_b200.h).

Loading fails loudly when the library is missing: there is no Python or CPU
fallback for any operation of this package.
"""
from __future__ import annotations

import ctypes as ct
import os

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "libtierkv_b200.so")

u8p = ct.POINTER(ct.c_uint8)
u32p = ct.POINTER(ct.c_uint32)
i32p = ct.POINTER(ct.c_int32)
u64p = ct.POINTER(ct.c_uint64)
szp = ct.POINTER(ct.c_size_t)
vp = ct.c_void_p
sz = ct.c_size_t


class ModelSpecC(ct.Structure):
    _fields_ = [("num_layers", ct.c_uint32), ("bytes_per_token_per_layer", ct.c_uint32),
                ("page_tokens", ct.c_uint32), ("vocab_size", ct.c_uint32), ("model_tag", ct.c_char_p)]


class PagedLayoutC(ct.Structure):
    _fields_ = [("base", ct.c_uint64), ("layer_base_dev", ct.c_void_p), ("page_stride", ct.c_uint64),
                ("plane_stride", ct.c_uint64), ("token_stride", ct.c_uint32), ("plane_bytes", ct.c_uint32),
                ("n_planes", ct.c_uint32), ("page_tokens", ct.c_uint32), ("bpt", ct.c_uint32),
                ("shared_table", ct.c_uint32)]


class XferDescC(ct.Structure):
    _fields_ = [("chunk", ct.c_uint64), ("layer_stride", ct.c_uint64), ("table_dev", ct.c_void_p),
                ("table_stride", ct.c_uint32), ("first_page", ct.c_uint32), ("n_tokens", ct.c_uint32),
                ("pad", ct.c_uint32)]


class AffinePlanC(ct.Structure):
    _fields_ = [("n_desc", ct.c_uint32), ("pages_per_desc", ct.c_uint32), ("last_tokens", ct.c_uint32),
                ("first_page", ct.c_uint32), ("table_dev", ct.c_void_p), ("table_stride", ct.c_uint32),
                ("pad", ct.c_uint32), ("chunk0", ct.c_uint64), ("chunk_stride", ct.c_uint64),
                ("layer_stride", ct.c_uint64)]


class ChainDescC(ct.Structure):
    _fields_ = [("token_off", ct.c_uint64), ("n_tokens", ct.c_uint32), ("out_first", ct.c_uint32),
                ("parent", ct.c_uint8 * 32)]


class ConnectorConfigC(ct.Structure):
    _fields_ = [("layerwise", ct.c_int), ("pin_stores", ct.c_int), ("staging_budget_bytes", ct.c_size_t),
                ("staging_depth", ct.c_uint32), ("load_zero_copy", ct.c_int), ("store_zero_copy", ct.c_int),
                ("store_ctas", ct.c_int),
                ("load_ctas", ct.c_int), ("engine_stream", ct.c_void_p), ("memo_entries", ct.c_size_t)]


class CodecItemC(ct.Structure):
    _fields_ = [("src_dev", ct.c_void_p), ("dst_dev", ct.c_void_p), ("bytes", ct.c_uint64)]


class PdRecordC(ct.Structure):
    _fields_ = [("addr", ct.c_uint64), ("bytes", ct.c_uint64), ("token_count", ct.c_uint32),
                ("first_token", ct.c_uint32)]


# name -> (restype, argtypes); the authoritative list of exported symbols.
SIGNATURES = {
    "tkv_last_error": (ct.c_char_p, []),
    "tkv_errc_name": (ct.c_char_p, [ct.c_int]),
    "tkv_build_info": (ct.c_char_p, []),
    "tkv_launch_count": (ct.c_uint64, []),
    "tkv_host_copy": (None, [vp, vp, ct.c_size_t]),
    "tkv_plan_tiles": (ct.c_int, [ct.c_void_p, ct.c_uint32, ct.c_uint32, ct.c_uint32, ct.c_uint32,
                                  ct.c_uint32, u32p, u32p]),
    "tkv_gather_layers": (ct.c_int, [ct.POINTER(PagedLayoutC), vp, vp, ct.c_uint32, ct.c_uint32, ct.c_uint32,
                                     ct.c_uint32, ct.c_uint32, ct.c_uint64, ct.c_int, vp]),
    "tkv_scatter_layers": (ct.c_int, [ct.POINTER(PagedLayoutC), vp, vp, ct.c_uint32, ct.c_uint32, ct.c_uint32,
                                      ct.c_uint32, ct.c_uint32, ct.c_uint64, ct.c_int, vp]),
    "tkv_affine_form": (ct.c_int, [vp, ct.c_uint32, ct.c_uint32, ct.POINTER(AffinePlanC)]),
    "tkv_gather_layers_affine": (ct.c_int, [ct.POINTER(PagedLayoutC), ct.POINTER(AffinePlanC), ct.c_uint32,
                                            ct.c_uint32, ct.c_int, vp]),
    "tkv_scatter_layers_affine": (ct.c_int, [ct.POINTER(PagedLayoutC), ct.POINTER(AffinePlanC), ct.c_uint32,
                                             ct.c_uint32, ct.c_int, vp]),
    "tkv_hash_chains": (ct.c_int, [vp, vp, ct.c_uint32, ct.c_uint32, ct.c_char_p, ct.c_uint32, vp, vp]),
    "tkv_synth_pages": (ct.c_int, [ct.POINTER(PagedLayoutC), vp, vp, ct.c_uint32, ct.c_uint64, ct.c_uint32,
                                   ct.c_uint32, ct.c_uint32, ct.c_uint32, vp]),
    "tkv_verify_pages": (ct.c_int, [ct.POINTER(PagedLayoutC), vp, vp, ct.c_uint32, ct.c_uint64, ct.c_uint32,
                                    ct.c_uint32, ct.c_uint32, ct.c_uint32, vp, vp]),
    "tkv_synth_chunk": (ct.c_int, [vp, ct.c_uint64, ct.c_uint32, ct.c_uint32, ct.c_uint32, ct.c_uint32, vp, vp]),
    "tkv_sm_copy": (ct.c_int, [vp, vp, ct.c_uint64, vp]),
    "tkv_ce_copy_pieces": (ct.c_int, [vp, vp, vp, ct.c_size_t, ct.c_int, vp]),
    "tkv_plan_copy_runs": (ct.c_size_t, [vp, vp, vp, ct.c_size_t, ct.c_size_t, vp, vp]),
    "tkv_ce_copy": (ct.c_int, [vp, vp, ct.c_uint64, vp]),
    "tkv_q8_blob_bytes": (ct.c_uint64, [ct.c_uint64]),
    "tkv_codec_plan": (ct.c_int, [vp, ct.c_uint32, u32p]),
    "tkv_q8_encode": (ct.c_int, [vp, vp, ct.c_uint32, ct.c_uint32, vp, vp]),
    "tkv_q8_encode_scratch_bytes": (ct.c_uint64, [ct.c_uint32]),
    "tkv_q8_decode": (ct.c_int, [vp, vp, ct.c_uint32, ct.c_uint32, vp]),
    "tkv_chunk_keys": (ct.c_int, [ct.c_char_p, sz, u32p, sz, u8p, szp]),
    "tkv_keychain_next": (ct.c_int, [ct.c_char_p, sz, u8p, u32p, sz, u8p]),
    "tkv_pages_create": (ct.c_int, [ct.POINTER(ModelSpecC), ct.c_uint32, ct.c_int, ct.POINTER(vp)]),
    "tkv_pages_destroy": (None, [vp]),
    "tkv_pages_alloc": (ct.c_int, [vp, ct.c_uint64, sz, u32p]),
    "tkv_pages_bind_layer": (ct.c_int, [vp, ct.c_uint64, ct.c_uint32, u32p, sz]),
    "tkv_pages_admit": (ct.c_int, [vp, ct.c_uint64, sz]),
    "tkv_pages_layer_pages": (sz, [vp, ct.c_uint64, ct.c_uint32, u32p, sz]),
    "tkv_pages_release": (sz, [vp, ct.c_uint64]),
    "tkv_pages_free_count": (sz, [vp]),
    "tkv_pages_allocated_count": (sz, [vp]),
    "tkv_pages_pool_pages": (sz, [vp]),
    "tkv_pages_mark_populated": (ct.c_int, [vp, ct.c_uint32, ct.c_uint32]),
    "tkv_pages_populated": (ct.c_int, [vp, ct.c_uint32]),
    "tkv_pages_gather": (ct.c_int, [vp, u32p, sz, ct.c_uint32, sz, u8p, sz]),
    "tkv_pages_scatter": (ct.c_int, [vp, u8p, sz, u32p, sz, ct.c_uint32, sz]),
    "tkv_pages_layout": (ct.c_int, [vp, ct.POINTER(PagedLayoutC)]),
    "tkv_pages_device_table": (ct.c_int, [vp, ct.c_uint64, vp, ct.POINTER(vp), u32p]),
    "tkv_pages_set_shard": (ct.c_int, [vp, ct.c_uint64]),
    "tkv_pages_compute": (ct.c_int, [vp, ct.c_uint64, vp, ct.c_uint32, ct.c_uint32, ct.c_uint32, ct.c_uint32, vp]),
    "tkv_pages_verify": (ct.c_int, [vp, ct.c_uint64, vp, ct.c_uint32, ct.c_uint32, ct.c_uint32, ct.c_uint32,
                                    vp, vp]),
    "tkv_store_create": (ct.c_int, [ct.POINTER(ModelSpecC), sz, sz, ct.POINTER(vp)]),
    "tkv_store_destroy": (None, [vp]),
    "tkv_store_put": (ct.c_int, [vp, u8p, ct.c_uint32, u8p, sz, ct.c_int]),
    "tkv_store_get": (ct.c_int, [vp, u8p, u8p, sz, szp]),
    "tkv_store_get_layer": (ct.c_int, [vp, u8p, ct.c_uint32, u8p, sz, szp]),
    "tkv_store_contains": (ct.c_int, [vp, u8p]),
    "tkv_store_pin": (ct.c_int, [vp, u8p, ct.c_int]),
    "tkv_store_clear": (ct.c_int, [vp, u8p, sz, szp, szp]),
    "tkv_store_stats": (ct.c_int, [vp, szp]),
    "tkv_store_verify_synth": (ct.c_int, [vp, u8p, vp, ct.c_uint64, ct.c_uint32, ct.c_uint64, vp, vp]),
    "tkv_model_tag_hash": (ct.c_int, [ct.c_char_p, u64p]),
    "tkv_store_export_record": (ct.c_int, [vp, u8p, ct.c_uint64, u8p, sz, szp]),
    "tkv_store_import_record": (ct.c_int, [vp, u8p, sz, ct.c_int]),
    "tkv_record_peek": (ct.c_int, [u8p, sz, u8p, u32p, u64p]),
    "tkv_connector_config_default": (None, [ct.POINTER(ConnectorConfigC)]),
    "tkv_connector_create": (ct.c_int, [vp, vp, ct.POINTER(ConnectorConfigC), ct.POINTER(vp)]),
    "tkv_connector_destroy": (None, [vp]),
    "tkv_connector_get_num_new_matched_tokens": (ct.c_int, [vp, ct.c_uint64, u32p, sz, szp]),
    "tkv_connector_lookup_batch": (ct.c_int, [vp, sz, u64p, ct.POINTER(u32p), szp, szp]),
    "tkv_connector_update_state_after_alloc": (ct.c_int, [vp, ct.c_uint64, sz, sz]),
    "tkv_connector_build_meta": (ct.c_int, [vp, sz, u64p, ct.POINTER(u32p), szp, ct.POINTER(vp)]),
    "tkv_connector_start_load_kv": (ct.c_int, [vp, vp]),
    "tkv_connector_wait_load_kv": (ct.c_int, [vp, vp, ct.c_uint32]),
    "tkv_connector_start_store_kv": (ct.c_int, [vp, vp]),
    "tkv_connector_wait_store_kv": (ct.c_int, [vp, vp, ct.c_uint32]),
    "tkv_connector_prefetch": (ct.c_int, [vp, u32p, sz]),
    "tkv_connector_drain_prefetch": (ct.c_int, [vp]),
    "tkv_connector_begin_decode": (ct.c_int, [vp, ct.c_uint64]),
    "tkv_connector_append_decode": (ct.c_int, [vp, ct.c_uint64, ct.c_uint32]),
    "tkv_connector_append_decode_batch": (ct.c_int, [vp, sz, u64p, u32p, ct.POINTER(ct.c_int)]),
    "tkv_connector_finish_query": (ct.c_int, [vp, ct.c_uint64, u8p, sz, szp]),
    "tkv_connector_staging_peak": (sz, [vp]),
    "tkv_connector_copy_runs": (None, [vp, u64p]),
    "tkv_connector_memo_stats": (ct.c_int, [vp, u64p]),
    "tkv_connector_debug_poison_memo": (ct.c_int, [vp]),
    "tkv_connector_hash_launches": (ct.c_uint64, [vp]),
    "tkv_connector_lookups_host_decided": (ct.c_uint64, [vp]),
    "tkv_connector_lookups_witnessed": (ct.c_uint64, [vp]),
    "tkv_meta_destroy": (None, [vp]),
    "tkv_meta_layerwise": (ct.c_int, [vp]),
    "tkv_meta_loaded_tokens": (sz, [vp, ct.c_uint64]),
    "tkv_meta_num_plans": (sz, [vp]),
    "tkv_meta_plan": (ct.c_int, [vp, sz, ct.c_int, u64p, u8p, sz, szp, u64p]),
    "tkv_meta_store_results": (ct.c_int, [vp, ct.c_uint64, ct.POINTER(ct.c_int), u8p, sz, szp]),
    "tkv_meta_timeline": (ct.c_int, [vp, ct.POINTER(ct.c_float), sz, szp]),
    "tkv_meta_origin_since": (ct.c_int, [vp, vp, ct.POINTER(ct.c_float)]),
    "tkv_pd_staging_create": (ct.c_int, [ct.POINTER(vp)]),
    "tkv_pd_staging_destroy": (None, [vp]),
    "tkv_pd_register": (ct.c_int, [vp, ct.c_uint64]),
    "tkv_pd_push": (ct.c_int, [vp, ct.c_uint64, ct.c_uint32, ct.c_int, ct.POINTER(PdRecordC)]),
    "tkv_pd_await": (ct.c_int, [vp, ct.c_uint64, ct.POINTER(PdRecordC), sz, szp]),
    "tkv_pd_cancel": (ct.c_int, [vp, ct.c_uint64]),
    "tkv_pd_registered": (sz, [vp]),
    "tkv_pd_send": (ct.c_int, [vp, ct.c_uint64, sz, sz, ct.c_uint64, ct.c_uint64, vp, ct.POINTER(PdRecordC), sz,
                               szp]),
    "tkv_pd_sender_begin": (ct.c_int, [vp, ct.c_uint64, sz, sz, ct.c_uint64, ct.c_uint64, ct.POINTER(vp)]),
    "tkv_pd_sender_layer": (ct.c_int, [vp, ct.c_uint32, vp]),
    "tkv_pd_sender_finish": (ct.c_int, [vp, ct.POINTER(PdRecordC), sz, szp]),
    "tkv_pd_sender_destroy": (None, [vp]),
    "tkv_pd_send_staged": (ct.c_int, [vp, ct.c_uint64, sz, sz, ct.c_uint64, ct.c_uint64, ct.c_uint64,
                                      ct.c_uint64, vp, ct.POINTER(PdRecordC), sz, szp]),
    "tkv_pd_land": (ct.c_int, [vp, ct.c_uint64, ct.POINTER(PdRecordC), sz, vp]),
    "tkv_enable_peer_access": (ct.c_int, [ct.c_int, ct.c_int]),
    "tkv_ipc_get_handle": (ct.c_int, [vp, u8p, ct.POINTER(ct.c_uint64)]),
    "tkv_ipc_open_handle": (ct.c_int, [u8p, ct.c_uint64, ct.POINTER(vp)]),
    "tkv_ipc_close": (ct.c_int, [vp, ct.c_uint64]),
}

_lib = None


class TkvError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"errc={code}: {msg}")
        self.code = code


def lib():
    """The loaded library (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2510_09665_b200._build` "
                "(there is no CPU fallback)")
        h = ct.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(h, name)
            f.restype = res
            f.argtypes = args
        _lib = h
    return _lib


def check(rc: int) -> int:
    if rc != 0:
        raise TkvError(rc, lib().tkv_last_error().decode(errors="replace"))
    return rc
