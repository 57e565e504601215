"""TEST INFRASTRUCTURE ONLY — the parity oracle for the tierkv hot path.

Two checkers live here, and nothing in ``paper_2510_09665_b200`` may import
either of them (tests/test_product_isolation.py enforces it):

* ``C`` — ctypes binding of ``liboracle.so``, our plain-C restatement of the
  reference arithmetic (tierkv_oracle.c: SHA-256 key chain, LPM, splitmix
  synth KV, page gather/scatter), each function citing the reference
  file:line it follows.
* ``Ref`` — ctypes binding of ``_ref/libtierkv_ref.so``: the UNMODIFIED
  reference sources compiled in place (oracle/Makefile) plus ``ref_shim.cpp``,
  which drives the reference's own public API (TieredStore, PagedKVStore,
  Connector, PdStaging). Present wherever it was built (this container, and
  the GPU box, where the prebuilt .so travels); tests skip when absent.

Parity pin: ``C`` is checked against SURVEY.md Appendix A and against the
fixtures in tests/golden/ produced by ``Ref`` (tests/golden/make_golden.py).
"""
from __future__ import annotations

import ctypes as ct
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_C = os.path.join(HERE, "liboracle.so")
LIB_REF = os.path.join(HERE, "_ref", "libtierkv_ref.so")

_u8p = ct.POINTER(ct.c_uint8)
_u32p = ct.POINTER(ct.c_uint32)
_u64p = ct.POINTER(ct.c_uint64)


def build(reference_root: str = "/root/reference/proj") -> None:
    """Build liboracle.so and, when the reference sources exist, _ref/."""
    targets = ["all"] if os.path.isdir(os.path.join(reference_root, "src")) else [LIB_C]
    subprocess.run(["make", "-s", "-C", HERE, f"REF={reference_root}", *targets], check=True)


def _ptr(a: np.ndarray, typ):
    return a.ctypes.data_as(typ)


def _tokens(tokens) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(tokens, dtype=np.uint32))


class _COracle:
    def __init__(self, path: str = LIB_C):
        if not os.path.exists(path):
            build()
        lib = ct.CDLL(path)
        lib.tkvo_sha256.argtypes = [_u8p, ct.c_size_t, _u8p]
        lib.tkvo_keychain_next.argtypes = [ct.c_char_p, ct.c_size_t, _u8p, _u32p, ct.c_size_t, _u8p]
        lib.tkvo_chunk_keys.argtypes = [_u32p, ct.c_size_t, ct.c_size_t, ct.c_char_p, ct.c_size_t, _u8p]
        lib.tkvo_chunk_keys.restype = ct.c_size_t
        lib.tkvo_longest_prefix_match.argtypes = [_u32p, ct.c_size_t, ct.c_size_t, ct.c_char_p,
                                                  ct.c_size_t, _u8p, ct.c_size_t]
        lib.tkvo_longest_prefix_match.restype = ct.c_size_t
        lib.tkvo_fnv1a64.argtypes = [_u8p, ct.c_size_t]
        lib.tkvo_fnv1a64.restype = ct.c_uint64
        lib.tkvo_splitmix64.argtypes = [ct.c_uint64]
        lib.tkvo_splitmix64.restype = ct.c_uint64
        lib.tkvo_model_seed.argtypes = [ct.c_char_p, ct.c_size_t]
        lib.tkvo_model_seed.restype = ct.c_uint64
        lib.tkvo_model_tag_hash.argtypes = [ct.c_char_p, ct.c_size_t]
        lib.tkvo_model_tag_hash.restype = ct.c_uint64
        lib.tkvo_synth_token_kv.argtypes = [ct.c_uint64, ct.c_uint32, ct.c_uint32, ct.c_uint64, _u8p, ct.c_size_t]
        lib.tkvo_synth_layer_kv.argtypes = [ct.c_uint64, _u32p, ct.c_size_t, ct.c_uint32, ct.c_uint64,
                                            ct.c_size_t, _u8p]
        lib.tkvo_synth_chunk.argtypes = [ct.c_uint64, _u32p, ct.c_size_t, ct.c_size_t, ct.c_uint32,
                                         ct.c_size_t, _u8p]
        lib.tkvo_q8_encode.argtypes = [_u8p, ct.c_size_t, _u8p]
        lib.tkvo_q8_encode.restype = ct.c_size_t
        lib.tkvo_q8_decode.argtypes = [_u8p, ct.c_size_t, _u8p]
        lib.tkvo_q8_decode.restype = ct.c_size_t
        lib.tkvo_gather_tokens.argtypes = [_u8p, ct.c_size_t, _u32p, ct.c_size_t, ct.c_size_t, ct.c_size_t, _u8p]
        lib.tkvo_scatter_tokens.argtypes = [_u8p, ct.c_size_t, _u32p, ct.c_size_t, ct.c_size_t, ct.c_size_t, _u8p]
        self.lib = lib

    def sha256(self, data: bytes) -> bytes:
        buf = np.frombuffer(bytes(data), dtype=np.uint8).copy()
        out = np.zeros(32, np.uint8)
        self.lib.tkvo_sha256(_ptr(buf, _u8p), buf.size, _ptr(out, _u8p))
        return out.tobytes()

    def keychain_next(self, tag: str, parent: bytes, tokens) -> bytes:
        t = _tokens(tokens)
        p = np.frombuffer(parent, dtype=np.uint8).copy()
        out = np.zeros(32, np.uint8)
        tb = tag.encode()
        self.lib.tkvo_keychain_next(tb, len(tb), _ptr(p, _u8p), _ptr(t, _u32p), t.size, _ptr(out, _u8p))
        return out.tobytes()

    def chunk_keys(self, tokens, chunk_size: int, tag: str) -> list[bytes]:
        t = _tokens(tokens)
        n_chunks = (t.size + chunk_size - 1) // chunk_size
        out = np.zeros(max(1, n_chunks) * 32, np.uint8)
        tb = tag.encode()
        n = self.lib.tkvo_chunk_keys(_ptr(t, _u32p), t.size, chunk_size, tb, len(tb), _ptr(out, _u8p))
        return [out[32 * i:32 * i + 32].tobytes() for i in range(n)]

    def longest_prefix_match(self, tokens, chunk_size: int, tag: str, digests) -> int:
        t = _tokens(tokens)
        d = np.frombuffer(b"".join(digests) or b"\0", dtype=np.uint8).copy()
        tb = tag.encode()
        return int(self.lib.tkvo_longest_prefix_match(_ptr(t, _u32p), t.size, chunk_size, tb, len(tb),
                                                      _ptr(d, _u8p), len(digests)))

    def fnv1a64(self, data) -> int:
        b = np.frombuffer(bytes(data), dtype=np.uint8).copy() if not isinstance(data, np.ndarray) else data
        return int(self.lib.tkvo_fnv1a64(_ptr(b, _u8p), b.size))

    def splitmix64(self, x: int) -> int:
        return int(self.lib.tkvo_splitmix64(x))

    def model_seed(self, tag: str) -> int:
        tb = tag.encode()
        return int(self.lib.tkvo_model_seed(tb, len(tb)))

    def model_tag_hash(self, tag: str) -> int:
        tb = tag.encode()
        return int(self.lib.tkvo_model_tag_hash(tb, len(tb)))

    def synth_token_kv(self, seed: int, token: int, layer: int, pos: int, bpt: int) -> np.ndarray:
        out = np.zeros(bpt, np.uint8)
        self.lib.tkvo_synth_token_kv(seed, token, layer, pos, _ptr(out, _u8p), bpt)
        return out

    def synth_layer_kv(self, seed: int, tokens, layer: int, first_pos: int, bpt: int) -> np.ndarray:
        t = _tokens(tokens)
        out = np.zeros(t.size * bpt, np.uint8)
        self.lib.tkvo_synth_layer_kv(seed, _ptr(t, _u32p), t.size, layer, first_pos, bpt, _ptr(out, _u8p))
        return out

    def synth_chunk(self, seed: int, prompt, start: int, n: int, num_layers: int, bpt: int) -> np.ndarray:
        """Layer-major chunk payload [L][n][bpt] (kv_chunk.hpp:12-36)."""
        t = _tokens(prompt)
        out = np.zeros(num_layers * n * bpt, np.uint8)
        self.lib.tkvo_synth_chunk(seed, _ptr(t, _u32p), start, n, num_layers, bpt, _ptr(out, _u8p))
        return out

    def q8_encode(self, payload: np.ndarray) -> np.ndarray:
        p = np.ascontiguousarray(payload, np.uint8)
        out = np.zeros(8 + p.size // 2 + (p.size & 1), np.uint8)
        n = self.lib.tkvo_q8_encode(_ptr(p, _u8p), p.size, _ptr(out, _u8p))
        return out[:n]

    def q8_decode(self, blob: np.ndarray) -> np.ndarray | None:
        b = np.ascontiguousarray(blob, np.uint8)
        if b.size < 8:
            return None
        length = int(b[:4].view(np.uint32)[0])
        out = np.zeros(max(1, length), np.uint8)
        n = self.lib.tkvo_q8_decode(_ptr(b, _u8p), b.size, _ptr(out, _u8p))
        if n != length or (n == 0 and b.size != 8):  # malformed blob
            return None
        return out[:length]

    def gather_tokens(self, pool: np.ndarray, page_bytes: int, pages, bpt: int, token_count: int) -> np.ndarray:
        p = _tokens(pages)
        out = np.zeros(token_count * bpt, np.uint8)
        self.lib.tkvo_gather_tokens(_ptr(pool, _u8p), page_bytes, _ptr(p, _u32p), p.size, bpt,
                                    token_count, _ptr(out, _u8p))
        return out

    def scatter_tokens(self, pool: np.ndarray, page_bytes: int, pages, bpt: int, token_count: int,
                       data: np.ndarray) -> None:
        p = _tokens(pages)
        d = np.ascontiguousarray(data, dtype=np.uint8)
        self.lib.tkvo_scatter_tokens(_ptr(pool, _u8p), page_bytes, _ptr(p, _u32p), p.size, bpt,
                                     token_count, _ptr(d, _u8p))


_c_singleton: _COracle | None = None


def C() -> _COracle:
    global _c_singleton
    if _c_singleton is None:
        _c_singleton = _COracle()
    return _c_singleton


def ref_available() -> bool:
    return os.path.exists(LIB_REF)


from .refshim import Ref, RefEngine  # noqa: E402  (re-export)
