"""TEST INFRASTRUCTURE ONLY — ctypes driver for the unmodified reference
(oracle/_ref/libtierkv_ref.so, built by oracle/Makefile from
/root/reference/proj/src plus oracle/ref_shim.cpp).

``RefEngine`` exposes the reference engine stack (TieredStore + PagedKVStore +
Connector, include/tierkv/connector.hpp:74-152) with the same method names as
the product's ``paper_2510_09665_b200.Engine``, so one scenario script can run
against both and compare outputs byte for byte.
"""
from __future__ import annotations

import ctypes as ct
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_REF = os.path.join(HERE, "_ref", "libtierkv_ref.so")

_u8p = ct.POINTER(ct.c_uint8)
_u32p = ct.POINTER(ct.c_uint32)
_u64p = ct.POINTER(ct.c_uint64)
_sz = ct.c_size_t
_vp = ct.c_void_p


def _tokens(tokens) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(tokens, dtype=np.uint32))


class _Ref:
    def __init__(self, path: str = LIB_REF):
        lib = ct.CDLL(path)
        sig = {
            "ref_chunk_keys": (_sz, [_u32p, _sz, _sz, ct.c_char_p, _u8p]),
            "ref_keychain_next": (None, [_u8p, ct.c_uint32, _u32p, _sz, _sz, ct.c_char_p, _u8p]),
            "ref_longest_prefix_match": (_sz, [_u32p, _sz, _sz, ct.c_char_p, _u8p, _sz]),
            "ref_sha256": (None, [_u8p, _sz, _u8p]),
            "ref_model_tag_hash": (ct.c_uint64, [ct.c_char_p]),
            "ref_fnv1a64": (ct.c_uint64, [_u8p, _sz]),
            "ref_model_seed": (ct.c_uint64, [ct.c_char_p]),
            "ref_synth_layer_kv": (None, [ct.c_uint64, _u32p, _sz, ct.c_uint32, ct.c_uint64, ct.c_uint32, _u8p]),
            "ref_encode_record": (_sz, [ct.c_char_p, _u8p, ct.c_uint32, ct.c_uint32, ct.c_uint32, _u8p, _u8p]),
            "ref_parse_record": (ct.c_int, [_u8p, _sz, _u8p]),
            "ref_q8_encode": (_sz, [_u8p, _sz, _u8p]),
            "ref_q8_decode": (_sz, [_u8p, _sz, _u8p, ct.POINTER(ct.c_int)]),
            "ref_engine_create": (_vp, [ct.c_uint32, ct.c_uint32, ct.c_uint32, ct.c_char_p, _sz, _sz, _sz,
                                        ct.c_uint32, ct.c_int, _sz, _sz, ct.c_int]),
            "ref_engine_destroy": (None, [_vp]),
            "ref_bind_pages": (ct.c_int, [_vp, ct.c_uint64, _sz]),
            "ref_release_query": (_sz, [_vp, ct.c_uint64]),
            "ref_free_pages": (_sz, [_vp]),
            "ref_compute_range": (None, [_vp, ct.c_uint64, _u32p, _sz, _sz]),
            "ref_gather_layer": (ct.c_int, [_vp, ct.c_uint64, ct.c_uint32, _sz, _u8p]),
            "ref_match": (_sz, [_vp, ct.c_uint64, _u32p, _sz]),
            "ref_update_alloc": (ct.c_int, [_vp, ct.c_uint64, _sz, _sz]),
            "ref_build_meta": (ct.c_int, [_vp, _sz, _u64p, ct.POINTER(_u32p), ct.POINTER(_sz)]),
            "ref_start_load": (ct.c_int, [_vp, ct.c_int]),
            "ref_wait_load": (ct.c_int, [_vp, ct.c_int, ct.c_uint32]),
            "ref_start_store": (ct.c_int, [_vp, ct.c_int]),
            "ref_wait_store": (ct.c_int, [_vp, ct.c_int, ct.c_uint32]),
            "ref_meta_layerwise": (ct.c_int, [_vp, ct.c_int]),
            "ref_meta_loaded": (_sz, [_vp, ct.c_int, ct.c_uint64]),
            "ref_meta_drop": (None, [_vp, ct.c_int]),
            "ref_meta_plan": (_sz, [_vp, ct.c_int, _sz, ct.c_int, _u64p, _u8p, _sz, _u64p]),
            "ref_meta_store_results": (_sz, [_vp, ct.c_int, ct.c_uint64, ct.POINTER(ct.c_int), _u8p, _sz]),
            "ref_finish_query": (ct.c_int, [_vp, ct.c_uint64]),
            "ref_begin_decode": (ct.c_int, [_vp, ct.c_uint64]),
            "ref_append_decode": (ct.c_int, [_vp, ct.c_uint64, ct.c_uint32, _sz]),
            "ref_finish_query_keys": (_sz, [_vp, ct.c_uint64, _u8p, _sz, ct.POINTER(ct.c_int)]),
            "ref_store_contains": (ct.c_int, [_vp, _u8p]),
            "ref_store_get": (_sz, [_vp, _u8p, _u8p, _sz]),
            "ref_store_clear": (_sz, [_vp, _u8p]),
            "ref_store_entries": (_sz, [_vp]),
            "ref_store_put": (ct.c_int, [_vp, _u8p, ct.c_uint32, _u8p, _sz, ct.c_int]),
            "ref_store_pin": (ct.c_int, [_vp, _u8p, ct.c_int]),
            "ref_store_get_layer": (ct.c_int, [_vp, _u8p, ct.c_uint32, _u8p, _sz, ct.POINTER(_sz)]),
            "ref_store_clear_n": (ct.c_int, [_vp, _u8p, ct.POINTER(_sz), ct.POINTER(_sz)]),
            "ref_store_stats": (None, [_vp, ct.POINTER(_sz)]),
            "ref_seed_store": (ct.c_int, [_vp, _u32p, _sz]),
            "ref_staging_peak": (ct.c_int64, [_vp]),
            "ref_staging_refs": (ct.c_int64, [_vp]),
            "ref_pd_create": (_vp, []),
            "ref_pd_destroy": (None, [_vp]),
            "ref_pd_register": (ct.c_int, [_vp, ct.c_uint64]),
            "ref_pd_push": (ct.c_int, [_vp, ct.c_uint64, ct.c_uint32, ct.c_int, _u8p, _sz]),
            "ref_pd_cancel": (ct.c_int, [_vp, ct.c_uint64]),
            "ref_pd_await": (ct.c_int, [_vp, ct.c_uint64, _u8p, _sz, ct.POINTER(_sz)]),
        }
        for name, (res, args) in sig.items():
            f = getattr(lib, name)
            f.restype = res
            f.argtypes = args
        self.lib = lib

    def chunk_keys(self, tokens, chunk_size: int, tag: str) -> list[bytes]:
        t = _tokens(tokens)
        out = np.zeros(max(1, (t.size + chunk_size - 1) // chunk_size) * 32, np.uint8)
        n = self.lib.ref_chunk_keys(t.ctypes.data_as(_u32p), t.size, chunk_size, tag.encode(),
                                    out.ctypes.data_as(_u8p))
        return [out[32 * i:32 * i + 32].tobytes() for i in range(n)]

    def keychain_next(self, tag: str, parent: bytes, index: int, tokens, chunk_size: int) -> bytes:
        t = _tokens(tokens)
        p = np.frombuffer(parent, np.uint8).copy()
        out = np.zeros(32, np.uint8)
        self.lib.ref_keychain_next(p.ctypes.data_as(_u8p), index, t.ctypes.data_as(_u32p), t.size,
                                   chunk_size, tag.encode(), out.ctypes.data_as(_u8p))
        return out.tobytes()

    def longest_prefix_match(self, tokens, chunk_size: int, tag: str, digests) -> int:
        t = _tokens(tokens)
        d = np.frombuffer(b"".join(digests) or b"\0", np.uint8).copy()
        return int(self.lib.ref_longest_prefix_match(t.ctypes.data_as(_u32p), t.size, chunk_size,
                                                     tag.encode(), d.ctypes.data_as(_u8p), len(digests)))

    def sha256(self, data: bytes) -> bytes:
        b = np.frombuffer(bytes(data) or b"\0", np.uint8).copy()
        out = np.zeros(32, np.uint8)
        self.lib.ref_sha256(b.ctypes.data_as(_u8p), len(data), out.ctypes.data_as(_u8p))
        return out.tobytes()

    def model_seed(self, tag: str) -> int:
        return int(self.lib.ref_model_seed(tag.encode()))

    def model_tag_hash(self, tag: str) -> int:
        return int(self.lib.ref_model_tag_hash(tag.encode()))

    def fnv1a64(self, data: np.ndarray) -> int:
        d = np.ascontiguousarray(data, np.uint8)
        return int(self.lib.ref_fnv1a64(d.ctypes.data_as(_u8p), d.size))

    def synth_layer_kv(self, seed: int, tokens, layer: int, first_pos: int, bpt: int) -> np.ndarray:
        t = _tokens(tokens)
        out = np.zeros(t.size * bpt, np.uint8)
        self.lib.ref_synth_layer_kv(seed, t.ctypes.data_as(_u32p), t.size, layer, first_pos, bpt,
                                    out.ctypes.data_as(_u8p))
        return out

    def encode_record(self, tag: str, digest: bytes, token_count: int, layers: int, bpt: int,
                      payload: np.ndarray) -> np.ndarray:
        p = np.ascontiguousarray(payload, np.uint8)
        d = np.frombuffer(digest, np.uint8).copy()
        out = np.zeros(54 + p.size + 8, np.uint8)  # kChunkHeaderBytes = 54 (chunk_file.hpp:18)
        n = self.lib.ref_encode_record(tag.encode(), d.ctypes.data_as(_u8p), token_count, layers, bpt,
                                       p.ctypes.data_as(_u8p), out.ctypes.data_as(_u8p))
        return out[:n]

    def parse_record(self, rec: np.ndarray, payload_bytes: int):
        r = np.ascontiguousarray(rec, np.uint8)
        out = np.zeros(max(1, payload_bytes), np.uint8)
        code = self.lib.ref_parse_record(r.ctypes.data_as(_u8p), r.size, out.ctypes.data_as(_u8p))
        return code, out[:payload_bytes]

    def q8_encode(self, payload: np.ndarray) -> np.ndarray:
        p = np.ascontiguousarray(payload, np.uint8)
        out = np.zeros(8 + p.size // 2 + (p.size & 1), np.uint8)
        n = self.lib.ref_q8_encode(p.ctypes.data_as(_u8p), p.size, out.ctypes.data_as(_u8p))
        return out[:n]

    def q8_decode(self, blob: np.ndarray):
        """(payload or None, Errc code)."""
        b = np.ascontiguousarray(blob, np.uint8)
        length = int(b[:4].view(np.uint32)[0]) if b.size >= 4 else 0
        out = np.zeros(max(1, length), np.uint8)
        code = ct.c_int(0)
        n = self.lib.ref_q8_decode(b.ctypes.data_as(_u8p), b.size, out.ctypes.data_as(_u8p), ct.byref(code))
        return (out[:n] if code.value == 0 else None), code.value


_ref_singleton: _Ref | None = None


def Ref() -> _Ref:
    global _ref_singleton
    if _ref_singleton is None:
        _ref_singleton = _Ref()
    return _ref_singleton


class RefEngine:
    """Reference TieredStore + PagedKVStore + Connector (one engine stack)."""

    def __init__(self, num_layers: int, bpt: int, page_tokens: int, tag: str, chunk_size: int,
                 ram_slots: int, num_pages: int, layerwise: bool = True,
                 staging_budget: int = 64 << 20, io_threads: int = 2, store_io_threads: int = 4,
                 pin_stores: bool = False):
        self.r = Ref()
        self.lib = self.r.lib
        self.num_layers, self.bpt, self.page_tokens = num_layers, bpt, page_tokens
        self.tag, self.chunk_size = tag, chunk_size
        ram = ram_slots * num_layers * chunk_size * bpt
        self.h = self.lib.ref_engine_create(num_layers, bpt, page_tokens, tag.encode(), chunk_size, ram,
                                            store_io_threads, num_pages, int(layerwise), staging_budget,
                                            io_threads, int(pin_stores))
        self._keep = []
        self._prompt_len: dict[int, int] = {}
        self._decode_pos: dict[int, int] = {}

    def close(self):
        if self.h:
            self.lib.ref_engine_destroy(self.h)
            self.h = None

    def __del__(self):
        self.close()

    # --- engine-side helpers (test_connector.cpp:101-178) ---
    def bind_pages(self, qid: int, tokens: int) -> int:
        return self.lib.ref_bind_pages(self.h, qid, tokens)

    def release_query(self, qid: int) -> int:
        return self.lib.ref_release_query(self.h, qid)

    def free_page_count(self) -> int:
        return self.lib.ref_free_pages(self.h)

    def compute_range(self, qid: int, prompt, start: int, end: int) -> None:
        t = _tokens(prompt)
        self.lib.ref_compute_range(self.h, qid, t.ctypes.data_as(_u32p), start, end)

    def gather_layer(self, qid: int, layer: int, n: int) -> np.ndarray:
        out = np.zeros(n * self.bpt, np.uint8)
        rc = self.lib.ref_gather_layer(self.h, qid, layer, n, out.ctypes.data_as(_u8p))
        if rc:
            raise RuntimeError(f"gather failed errc={rc}")
        return out

    def seed_store(self, prompt, n: int) -> None:
        t = _tokens(prompt)
        assert self.lib.ref_seed_store(self.h, t.ctypes.data_as(_u32p), n) == 0

    # --- connector (connector.hpp:96-119) ---
    def get_num_new_matched_tokens(self, qid: int, prompt) -> int:
        t = _tokens(prompt)
        return int(self.lib.ref_match(self.h, qid, t.ctypes.data_as(_u32p), t.size))

    def update_state_after_alloc(self, qid: int, blocks: int, ext: int) -> int:
        return self.lib.ref_update_alloc(self.h, qid, blocks, ext)

    def build_connector_meta(self, queries) -> int:
        ids = (ct.c_uint64 * len(queries))(*[q for q, _ in queries])
        arrs = [_tokens(p) for _, p in queries]
        self._keep.append(arrs)
        for (q, _), a in zip(queries, arrs):
            self._prompt_len[q] = a.size
        ptrs = (_u32p * len(queries))(*[a.ctypes.data_as(_u32p) for a in arrs])
        lens = (_sz * len(queries))(*[a.size for a in arrs])
        return self.lib.ref_build_meta(self.h, len(queries), ids, ptrs, lens)

    def start_load_kv(self, m: int) -> int:
        return self.lib.ref_start_load(self.h, m)

    def wait_load_kv(self, m: int, layer: int) -> int:
        return self.lib.ref_wait_load(self.h, m, layer)

    def start_store_kv(self, m: int) -> int:
        return self.lib.ref_start_store(self.h, m)

    def wait_store_kv(self, m: int, layer: int) -> int:
        return self.lib.ref_wait_store(self.h, m, layer)

    def meta_layerwise(self, m: int) -> bool:
        return bool(self.lib.ref_meta_layerwise(self.h, m))

    def loaded_tokens(self, m: int, qid: int) -> int:
        return int(self.lib.ref_meta_loaded(self.h, m, qid))

    def plan(self, m: int, qi: int, kind: str):
        """[(start, end, record_tokens, chunk_index, digest)] and matched."""
        k = 0 if kind == "load" else 1
        cap = 4096
        spans = np.zeros(4 * cap, np.uint64)
        dig = np.zeros(32 * cap, np.uint8)
        matched = ct.c_uint64(0)
        n = self.lib.ref_meta_plan(self.h, m, qi, k, spans.ctypes.data_as(_u64p), dig.ctypes.data_as(_u8p),
                                   cap, ct.byref(matched))
        out = [(int(spans[4 * i]), int(spans[4 * i + 1]), int(spans[4 * i + 2]), int(spans[4 * i + 3]),
                dig[32 * i:32 * i + 32].tobytes()) for i in range(n)]
        return out, int(matched.value)

    def store_results(self, m: int, qid: int):
        cap = 4096
        codes = (ct.c_int * cap)()
        dig = np.zeros(32 * cap, np.uint8)
        n = self.lib.ref_meta_store_results(self.h, m, qid, codes, dig.ctypes.data_as(_u8p), cap)
        return [(dig[32 * i:32 * i + 32].tobytes(), int(codes[i])) for i in range(n)]

    def finish_query(self, qid: int) -> int:
        self._decode_pos.pop(qid, None)
        return self.lib.ref_finish_query(self.h, qid)

    # --- decode storing (connector.hpp:116-119) ---
    def begin_decode(self, qid: int) -> int:
        rc = self.lib.ref_begin_decode(self.h, qid)
        if rc == 0:
            self._decode_pos[qid] = self._prompt_len.get(qid, 0)
        return rc

    def append_decode(self, qid: int, token: int) -> int:
        pos = self._decode_pos.get(qid, 0)
        rc = self.lib.ref_append_decode(self.h, qid, token, pos)
        if rc == 0:
            self._decode_pos[qid] = pos + 1
        return rc

    def finish_query_keys(self, qid: int):
        cap = 4096
        dig = np.zeros(32 * cap, np.uint8)
        code = ct.c_int(0)
        n = self.lib.ref_finish_query_keys(self.h, qid, dig.ctypes.data_as(_u8p), cap, ct.byref(code))
        self._decode_pos.pop(qid, None)
        return [dig[32 * i:32 * i + 32].tobytes() for i in range(n)], code.value

    def drop_meta(self, m: int) -> None:
        self.lib.ref_meta_drop(self.h, m)

    # --- store (store.hpp:153-171) ---
    def contains(self, digest: bytes) -> bool:
        d = np.frombuffer(digest, np.uint8).copy()
        return bool(self.lib.ref_store_contains(self.h, d.ctypes.data_as(_u8p)))

    def store_get(self, digest: bytes) -> np.ndarray | None:
        d = np.frombuffer(digest, np.uint8).copy()
        n = self.lib.ref_store_get(self.h, d.ctypes.data_as(_u8p), None, 0)
        if n == 0:
            return None
        out = np.zeros(n, np.uint8)
        self.lib.ref_store_get(self.h, d.ctypes.data_as(_u8p), out.ctypes.data_as(_u8p), n)
        return out

    def store_clear(self, digest: bytes) -> int:
        d = np.frombuffer(digest, np.uint8).copy()
        return int(self.lib.ref_store_clear(self.h, d.ctypes.data_as(_u8p)))

    def store_entries(self) -> int:
        return int(self.lib.ref_store_entries(self.h))

    def store_put(self, digest: bytes, token_count: int, payload: np.ndarray, pin: bool = False) -> int:
        d, p = np.frombuffer(digest, np.uint8).copy(), np.ascontiguousarray(payload, dtype=np.uint8)
        return int(self.lib.ref_store_put(self.h, d.ctypes.data_as(_u8p), token_count, p.ctypes.data_as(_u8p),
                                          p.size, int(pin)))

    def store_pin(self, digest: bytes, on: bool) -> int:
        d = np.frombuffer(digest, np.uint8).copy()
        return int(self.lib.ref_store_pin(self.h, d.ctypes.data_as(_u8p), int(on)))

    def store_get_layer(self, digest: bytes, layer: int):
        d = np.frombuffer(digest, np.uint8).copy()
        n = _sz(0)
        rc = self.lib.ref_store_get_layer(self.h, d.ctypes.data_as(_u8p), layer, None, 0, ct.byref(n))
        if rc:
            return int(rc), None
        out = np.zeros(n.value, np.uint8)
        self.lib.ref_store_get_layer(self.h, d.ctypes.data_as(_u8p), layer, out.ctypes.data_as(_u8p), n.value,
                                     ct.byref(n))
        return 0, out

    def store_clear_n(self, digest: bytes):
        d = np.frombuffer(digest, np.uint8).copy()
        removed, refused = _sz(0), _sz(0)
        self.lib.ref_store_clear_n(self.h, d.ctypes.data_as(_u8p), ct.byref(removed), ct.byref(refused))
        return removed.value, refused.value

    def store_stats(self):
        out = (_sz * 4)()
        self.lib.ref_store_stats(self.h, out)
        return tuple(int(x) for x in out)

    def staging_peak(self) -> int:
        return int(self.lib.ref_staging_peak(self.h))

    def staging_refs(self) -> int:
        return int(self.lib.ref_staging_refs(self.h))
