"""Python face of the B200 path: thin wrappers over the C-ABI objects.

``Engine`` bundles one PagedKVStore (device pages), one TieredStore (pinned
host tier) and one Connector, with the same method names and return
conventions as ``oracle.RefEngine`` (the reference engine stack) so that a
test scenario can be run against both and compared. Connector calls return
the reference's Errc codes as ints; everything else raises TkvError.

PyTorch is used only as plumbing: device buffers for prompt tokens and the
engine stream handle.
"""
from __future__ import annotations

import ctypes as ct

import numpy as np
import torch

from ._lib import (ChainDescC, ConnectorConfigC, ModelSpecC, PagedLayoutC, PdRecordC, XferDescC, check,
                   lib, u8p, u32p, u64p)

__all__ = ["Engine", "chunk_keys", "keychain_next", "PagedLayoutC", "XferDescC", "ChainDescC",
           "plan_tiles", "hash_chains", "ErrcOK"]

ErrcOK = 0


def _tokens(tokens) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(tokens, dtype=np.uint32))


def _u8(b: bytes) -> np.ndarray:
    return np.frombuffer(b, dtype=np.uint8).copy()


def chunk_keys(tokens, chunk_size: int, tag: str) -> list[bytes]:
    """Chunk keys of one sequence, computed by the K3 device kernel."""
    t = _tokens(tokens)
    n_chunks = (t.size + chunk_size - 1) // chunk_size
    out = np.zeros(max(1, n_chunks) * 32, np.uint8)
    n = ct.c_size_t(0)
    check(lib().tkv_chunk_keys(tag.encode(), chunk_size, t.ctypes.data_as(u32p), t.size,
                               out.ctypes.data_as(u8p), ct.byref(n)))
    return [out[32 * i:32 * i + 32].tobytes() for i in range(n.value)]


def keychain_next(tag: str, chunk_size: int, parent: bytes, tokens) -> bytes:
    t = _tokens(tokens)
    p = _u8(parent)
    out = np.zeros(32, np.uint8)
    check(lib().tkv_keychain_next(tag.encode(), chunk_size, p.ctypes.data_as(u8p), t.ctypes.data_as(u32p),
                                  t.size, out.ctypes.data_as(u8p)))
    return out.tobytes()


def plan_tiles(descs: list[XferDescC], page_tokens: int, page_bytes: int, n_layers: int,
               pages_per_tile: int = 0):
    """Host tile prefix for a K1/K2 launch: (tile_base uint32 array, ppt)."""
    arr = (XferDescC * max(1, len(descs)))(*descs)
    tb = np.zeros(len(descs) + 1, np.uint32)
    ppt = ct.c_uint32(0)
    check(lib().tkv_plan_tiles(ct.cast(arr, ct.c_void_p), len(descs), page_tokens, page_bytes,
                               pages_per_tile, n_layers, tb.ctypes.data_as(u32p), ct.byref(ppt)))
    return tb, ppt.value


def hash_chains(tokens_dev: torch.Tensor, chains_dev: torch.Tensor, n_chains: int, chunk_size: int,
                tag: str, out_dev: torch.Tensor, stream=None) -> None:
    s = stream.cuda_stream if stream is not None else torch.cuda.current_stream().cuda_stream
    tb = tag.encode()
    check(lib().tkv_hash_chains(tokens_dev.data_ptr(), chains_dev.data_ptr(), n_chains, chunk_size, tb,
                                len(tb), out_dev.data_ptr(), s))


class Engine:
    """Device pages + pinned host tier + connector (one engine stack)."""

    def __init__(self, num_layers: int, bpt: int, page_tokens: int, tag: str, chunk_size: int,
                 ram_slots: int, num_pages: int, layerwise: bool = True, staging_budget: int = 64 << 20,
                 io_threads: int = 2, store_io_threads: int = 4, pin_stores: bool = False,
                 staging_depth: int = 2, load_zero_copy: bool = False, store_zero_copy: bool = False,
                 store_ctas: int = 0,
                 load_ctas: int = 0, device: int = 0, stream: torch.cuda.Stream | None = None,
                 memo_entries: int | None = None, shard_offset: int = 0):
        del io_threads, store_io_threads  # host thread pools do not exist on this path
        self.L = lib()
        self.num_layers, self.bpt, self.page_tokens = num_layers, bpt, page_tokens
        self.tag, self.chunk_size = tag, chunk_size
        self.device = device
        torch.cuda.set_device(device)
        self.stream = stream
        self._tag_b = tag.encode()
        spec = ModelSpecC(num_layers, bpt, page_tokens, 32000, self._tag_b)
        self.pages = ct.c_void_p()
        self.store = ct.c_void_p()
        self.conn = ct.c_void_p()
        check(self.L.tkv_pages_create(ct.byref(spec), num_pages, device, ct.byref(self.pages)))
        if shard_offset:  # TP head shard: compute/verify produce this slice of the full row
            check(self.L.tkv_pages_set_shard(self.pages, shard_offset))
        ram = ram_slots * num_layers * chunk_size * bpt
        check(self.L.tkv_store_create(ct.byref(spec), chunk_size, ram, ct.byref(self.store)))
        cfg = ConnectorConfigC()
        self.L.tkv_connector_config_default(ct.byref(cfg))
        cfg.layerwise = int(layerwise)
        cfg.pin_stores = int(pin_stores)
        cfg.staging_budget_bytes = staging_budget
        cfg.staging_depth = staging_depth
        cfg.load_zero_copy = int(load_zero_copy)
        cfg.store_zero_copy = int(store_zero_copy)
        if store_ctas:
            cfg.store_ctas = store_ctas
        cfg.load_ctas = load_ctas
        cfg.engine_stream = self.stream_handle
        if memo_entries is not None:
            cfg.memo_entries = memo_entries
        check(self.L.tkv_connector_create(self.store, self.pages, ct.byref(cfg), ct.byref(self.conn)))
        self._metas: list[ct.c_void_p | None] = []
        self._dev_prompts: dict[int, torch.Tensor] = {}
        self._host_prompts: dict[int, np.ndarray] = {}
        self._prompt_src: dict[int, object] = {}
        self._host_tensors: dict[int, torch.Tensor] = {}
        self._retired_hosts: list = []
        self._mism = torch.zeros(1, dtype=torch.int64, device=f"cuda:{device}")

    @property
    def stream_handle(self):
        return self.stream.cuda_stream if self.stream is not None else None

    def close(self):
        if getattr(self, "conn", None):
            for i in range(len(self._metas)):
                self.drop_meta(i)
            self.L.tkv_connector_destroy(self.conn)
            self.conn = None
            self.L.tkv_store_destroy(self.store)
            self.L.tkv_pages_destroy(self.pages)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def synchronize(self):
        torch.cuda.synchronize(self.device)

    # --- engine-side helpers (mirror oracle.RefEngine) ---
    def bind_pages(self, qid: int, tokens: int) -> int:
        """Pages for `tokens`, bound per layer (SimEngine::admit)."""
        return self.L.tkv_pages_admit(self.pages, qid, tokens)

    def layer_pages(self, qid: int, layer: int) -> np.ndarray:
        n = self.L.tkv_pages_layer_pages(self.pages, qid, layer, None, 0)
        out = np.zeros(max(1, n), np.uint32)
        self.L.tkv_pages_layer_pages(self.pages, qid, layer, out.ctypes.data_as(u32p), n)
        return out[:n]

    def release_query(self, qid: int, sync: bool = True) -> int:
        """Free the query's pages. sync=False: the caller guarantees the
        query's transfers finished (its final store wait returned)."""
        if sync:
            self.synchronize()
        self._dev_prompts.pop(qid, None)
        self._host_prompts.pop(qid, None)
        self._prompt_src.pop(qid, None)
        self._retire_host(qid)
        return self.L.tkv_pages_release(self.pages, qid)

    def free_page_count(self) -> int:
        return self.L.tkv_pages_free_count(self.pages)

    def dev_prompt(self, qid: int, prompt) -> torch.Tensor:
        if self._prompt_src.get(qid) is prompt:  # same object as last call: no compare, no copy
            return self._dev_prompts[qid]
        t = _tokens(prompt)
        cur = self._dev_prompts.get(qid)
        self._prompt_src[qid] = prompt
        if cur is None or cur.numel() != t.size or not np.array_equal(self._host_prompts.get(qid), t):
            # Pinned host copy read by an SM-driven copy kernel on the engine
            # stream: a copy-engine upload would queue behind the layerwise KV
            # transfers already in flight. The pinned buffer
            # doubles as the host copy. A replaced buffer is retired with an
            # event and only returned to torch's pinned cache once the copy
            # reading it ran: torch records no use for a kernel's reads, and a
            # recycled block refilled by the host under a pending copy would
            # hand the engine another prompt's tokens.
            self._retire_host(qid)
            host = torch.empty(max(1, t.size), dtype=torch.int32, pin_memory=True)
            hv = host.numpy().view(np.uint32)[:t.size]
            hv[:] = t
            cur = torch.empty(max(1, t.size), dtype=torch.int32, device=f"cuda:{self.device}")[:t.size]
            check(self.L.tkv_sm_copy(host.data_ptr(), cur.data_ptr(), t.nbytes, self.stream_handle))
            if self.stream is not None:
                cur.record_stream(self.stream)
            self._host_prompts[qid] = hv
            self._host_tensors[qid] = host
            self._dev_prompts[qid] = cur
        return cur

    def _retire_host(self, qid: int) -> None:
        old = self._host_tensors.pop(qid, None)
        if old is not None:
            ev = torch.cuda.Event()
            ev.record(self.stream if self.stream is not None else torch.cuda.default_stream(self.device))
            self._retired_hosts.append((ev, old))
        self._retired_hosts = [(e, h) for e, h in self._retired_hosts if not e.query()]

    def compute_range(self, qid: int, prompt, start: int, end: int, layers=None) -> None:
        """Engine compute stand-in: synth KV for [start, end) into pages (K4)."""
        if end <= start:
            return
        toks = self.dev_prompt(qid, prompt)
        l0, l1 = layers if layers is not None else (0, self.num_layers)
        check(self.L.tkv_pages_compute(self.pages, qid, toks.data_ptr(), start, end, l0, l1,
                                       self.stream_handle))

    def verify_range(self, qid: int, prompt, start: int, end: int) -> int:
        """Device byte oracle: number of 8-byte words differing from synth."""
        toks = self.dev_prompt(qid, prompt)
        self._mism.zero_()
        self.synchronize()
        check(self.L.tkv_pages_verify(self.pages, qid, toks.data_ptr(), start, end, 0, self.num_layers,
                                      self._mism.data_ptr(), self.stream_handle))
        self.synchronize()
        return int(self._mism.item())

    def gather_layer(self, qid: int, layer: int, n: int) -> np.ndarray:
        pages = self.layer_pages(qid, layer)
        pages = np.ascontiguousarray(pages[:(n + self.page_tokens - 1) // self.page_tokens])
        out = np.zeros(max(1, n * self.bpt), np.uint8)
        check(self.L.tkv_pages_gather(self.pages, pages.ctypes.data_as(u32p), pages.size, layer, n,
                                      out.ctypes.data_as(u8p), n * self.bpt))
        return out[:n * self.bpt]

    def seed_store(self, prompt, n: int) -> None:
        """Store device-synthesized chunk payloads for prompt[0, n)."""
        t = _tokens(prompt)[:n]
        keys = chunk_keys(t, self.chunk_size, self.tag)
        dev = torch.from_numpy(t.view(np.int32)).to(f"cuda:{self.device}")
        seed = _model_seed(self.tag)
        for i, k in enumerate(keys):
            s = i * self.chunk_size
            cnt = min(self.chunk_size, n - s)
            buf = torch.empty(self.num_layers * cnt * self.bpt, dtype=torch.uint8, device=dev.device)
            check(self.L.tkv_synth_chunk(dev.data_ptr(), seed, s, cnt, self.num_layers, self.bpt,
                                         buf.data_ptr(), None))
            host = buf.cpu().numpy()
            d = _u8(k)
            check(self.L.tkv_store_put(self.store, d.ctypes.data_as(u8p), cnt, host.ctypes.data_as(u8p),
                                       host.size, 0))

    # --- connector ---
    def get_num_new_matched_tokens(self, qid: int, prompt) -> int:
        t = _tokens(prompt)
        # The engine receives the prompt at scheduling time; its device copy
        # goes up now, before this step's loads occupy the copy engines.
        self.dev_prompt(qid, t)
        m = ct.c_size_t(0)
        check(self.L.tkv_connector_get_num_new_matched_tokens(self.conn, qid, t.ctypes.data_as(u32p), t.size,
                                                              ct.byref(m)))
        return m.value

    def lookup_batch(self, qids, prompts) -> list[int]:
        arrs = [_tokens(p) for p in prompts]
        ids = (ct.c_uint64 * len(arrs))(*qids)
        ptrs = (u32p * len(arrs))(*[a.ctypes.data_as(u32p) for a in arrs])
        lens = (ct.c_size_t * len(arrs))(*[a.size for a in arrs])
        out = (ct.c_size_t * len(arrs))()
        check(self.L.tkv_connector_lookup_batch(self.conn, len(arrs), ids, ptrs, lens, out))
        return list(out)

    def update_state_after_alloc(self, qid: int, blocks: int, ext: int) -> int:
        return self.L.tkv_connector_update_state_after_alloc(self.conn, qid, blocks, ext)

    def build_connector_meta(self, queries) -> int:
        arrs = [_tokens(p) for _, p in queries]
        ids = (ct.c_uint64 * len(arrs))(*[q for q, _ in queries])
        ptrs = (u32p * len(arrs))(*[a.ctypes.data_as(u32p) for a in arrs])
        lens = (ct.c_size_t * len(arrs))(*[a.size for a in arrs])
        m = ct.c_void_p()
        check(self.L.tkv_connector_build_meta(self.conn, len(arrs), ids, ptrs, lens, ct.byref(m)))
        self._metas.append(m)
        return len(self._metas) - 1

    def start_load_kv(self, m: int) -> int:
        return self.L.tkv_connector_start_load_kv(self.conn, self._metas[m])

    def wait_load_kv(self, m: int, layer: int) -> int:
        return self.L.tkv_connector_wait_load_kv(self.conn, self._metas[m], layer)

    def start_store_kv(self, m: int) -> int:
        return self.L.tkv_connector_start_store_kv(self.conn, self._metas[m])

    def wait_store_kv(self, m: int, layer: int) -> int:
        return self.L.tkv_connector_wait_store_kv(self.conn, self._metas[m], layer)

    def meta_layerwise(self, m: int) -> bool:
        return bool(self.L.tkv_meta_layerwise(self._metas[m]))

    def loaded_tokens(self, m: int, qid: int) -> int:
        return int(self.L.tkv_meta_loaded_tokens(self._metas[m], qid))

    def plan(self, m: int, qi: int, kind: str):
        cap = 1 << 14
        spans = np.zeros(4 * cap, np.uint64)
        dig = np.zeros(32 * cap, np.uint8)
        n = ct.c_size_t(0)
        matched = ct.c_uint64(0)
        check(self.L.tkv_meta_plan(self._metas[m], qi, 0 if kind == "load" else 1, spans.ctypes.data_as(u64p),
                                   dig.ctypes.data_as(u8p), cap, ct.byref(n), ct.byref(matched)))
        out = [(int(spans[4 * i]), int(spans[4 * i + 1]), int(spans[4 * i + 2]), int(spans[4 * i + 3]),
                dig[32 * i:32 * i + 32].tobytes()) for i in range(n.value)]
        return out, int(matched.value)

    def store_results(self, m: int, qid: int):
        cap = 1 << 14
        codes = (ct.c_int * cap)()
        dig = np.zeros(32 * cap, np.uint8)
        n = ct.c_size_t(0)
        check(self.L.tkv_meta_store_results(self._metas[m], qid, codes, dig.ctypes.data_as(u8p), cap,
                                            ct.byref(n)))
        return [(dig[32 * i:32 * i + 32].tobytes(), int(codes[i])) for i in range(n.value)]

    def timeline(self, m: int) -> np.ndarray:
        """[layers, 5] ms: h2d done, load done, compute done, gathered, d2h done."""
        cap = 5 * self.num_layers
        out = (ct.c_float * cap)()
        n = ct.c_size_t(0)
        check(self.L.tkv_meta_timeline(self._metas[m], out, cap, ct.byref(n)))
        return np.array(out[:n.value], dtype=np.float32).reshape(-1, 5)

    def origin_since(self, m: int, event: torch.cuda.Event) -> float:
        """ms from a completed torch timing event to batch m's timeline origin."""
        ms = ct.c_float(-1.0)
        check(self.L.tkv_meta_origin_since(self._metas[m], ct.c_void_p(event.cuda_event), ct.byref(ms)))
        return ms.value

    def begin_decode(self, qid: int) -> int:
        return self.L.tkv_connector_begin_decode(self.conn, qid)

    def append_decode(self, qid: int, token: int) -> int:
        return self.L.tkv_connector_append_decode(self.conn, qid, token)

    def append_decode_batch(self, qids, tokens) -> list[int]:
        """One decode step for many queries in one call."""
        n = len(qids)
        q = (ct.c_uint64 * n)(*qids)
        t = (ct.c_uint32 * n)(*[int(x) for x in tokens])
        out = (ct.c_int * n)()
        check(self.L.tkv_connector_append_decode_batch(self.conn, n, q, t, out))
        return list(out)

    def finish_query(self, qid: int) -> int:
        keys, rc = self.finish_query_keys(qid)
        return rc

    def finish_query_keys(self, qid: int):
        cap = 4096
        dig = np.zeros(32 * cap, np.uint8)
        n = ct.c_size_t(0)
        rc = self.L.tkv_connector_finish_query(self.conn, qid, dig.ctypes.data_as(u8p), cap, ct.byref(n))
        return [dig[32 * i:32 * i + 32].tobytes() for i in range(n.value)], rc

    def drop_meta(self, m: int) -> None:
        h = self._metas[m]
        if h is not None:
            self.L.tkv_meta_destroy(h)
            self._metas[m] = None

    def staging_peak(self) -> int:
        return int(self.L.tkv_connector_staging_peak(self.conn))

    def copy_runs(self) -> tuple[int, int]:
        """(pieces, copies): host-tier chunk-layer pieces and the copy-engine copies they took."""
        out = (ct.c_uint64 * 2)()
        self.L.tkv_connector_copy_runs(self.conn, out)
        return int(out[0]), int(out[1])

    def lookups_host_decided(self) -> int:
        return int(self.L.tkv_connector_lookups_host_decided(self.conn))

    def lookups_witnessed(self) -> int:
        """Lookup rows the absence witness decided (absent, no SHA)."""
        return int(self.L.tkv_connector_lookups_witnessed(self.conn))

    def hash_launches(self) -> int:
        return int(self.L.tkv_connector_hash_launches(self.conn))

    def memo_stats(self) -> dict:
        out = (ct.c_uint64 * 5)()
        check(self.L.tkv_connector_memo_stats(self.conn, out))
        return {"hits": out[0], "misses": out[1], "capacity": out[2], "resets": out[3], "rehashes": out[4]}

    def debug_poison_memo(self) -> None:
        check(self.L.tkv_connector_debug_poison_memo(self.conn))

    # --- store ---
    def contains(self, digest: bytes) -> bool:
        d = _u8(digest)
        return bool(self.L.tkv_store_contains(self.store, d.ctypes.data_as(u8p)))

    def store_get(self, digest: bytes) -> np.ndarray | None:
        self.synchronize()
        d = _u8(digest)
        n = ct.c_size_t(0)
        rc = self.L.tkv_store_get(self.store, d.ctypes.data_as(u8p), None, 0, ct.byref(n))
        if rc:
            return None
        out = np.zeros(n.value, np.uint8)
        check(self.L.tkv_store_get(self.store, d.ctypes.data_as(u8p), out.ctypes.data_as(u8p), n.value,
                                   ct.byref(n)))
        return out

    def store_clear(self, digest: bytes) -> int:
        d = _u8(digest)
        removed = ct.c_size_t(0)
        refused = ct.c_size_t(0)
        check(self.L.tkv_store_clear(self.store, d.ctypes.data_as(u8p), 1, ct.byref(removed), ct.byref(refused)))
        return removed.value

    def store_entries(self) -> int:
        return self.store_stats()[0]

    # direct RAM-tier operations (same names and returns as oracle.RefEngine)
    def store_put(self, digest: bytes, token_count: int, payload: np.ndarray, pin: bool = False) -> int:
        d, p = _u8(digest), np.ascontiguousarray(payload, dtype=np.uint8)
        return int(self.L.tkv_store_put(self.store, d.ctypes.data_as(u8p), token_count, p.ctypes.data_as(u8p),
                                        p.size, int(pin)))

    def store_pin(self, digest: bytes, on: bool) -> int:
        return int(self.L.tkv_store_pin(self.store, _u8(digest).ctypes.data_as(u8p), int(on)))

    def store_get_layer(self, digest: bytes, layer: int):
        """(code, layer bytes or None)."""
        self.synchronize()
        d = _u8(digest)
        n = ct.c_size_t(0)
        rc = self.L.tkv_store_get_layer(self.store, d.ctypes.data_as(u8p), layer, None, 0, ct.byref(n))
        if rc:
            return int(rc), None
        out = np.zeros(n.value, np.uint8)
        check(self.L.tkv_store_get_layer(self.store, d.ctypes.data_as(u8p), layer, out.ctypes.data_as(u8p),
                                         n.value, ct.byref(n)))
        return 0, out

    def store_clear_n(self, digest: bytes):
        """(removed, refused)."""
        d = _u8(digest)
        removed, refused = ct.c_size_t(0), ct.c_size_t(0)
        check(self.L.tkv_store_clear(self.store, d.ctypes.data_as(u8p), 1, ct.byref(removed), ct.byref(refused)))
        return removed.value, refused.value

    def verify_stored(self, digest: bytes, prompt, start: int, shard_offset: int = 0) -> int | None:
        """Device byte oracle over one tier entry: mismatching 8-byte words of
        its pinned slot against synth for tokens [start, start + T) of
        `prompt` (the SMs read the slot over PCIe); None if absent."""
        t = _tokens(prompt)
        dev = torch.from_numpy(t.view(np.int32)).to(f"cuda:{self.device}")
        d = _u8(digest)
        self._mism.zero_()
        self.synchronize()
        rc = self.L.tkv_store_verify_synth(self.store, d.ctypes.data_as(u8p), dev.data_ptr(), _model_seed(self.tag),
                                           start, shard_offset, self._mism.data_ptr(), self.stream_handle)
        if rc == 1:  # not_found
            return None
        check(rc)
        return int(self._mism.item())

    def store_stats(self):
        """(entries, ram_slots_total, ram_slots_used, ram_entries)."""
        out = (ct.c_size_t * 4)()
        check(self.L.tkv_store_stats(self.store, out))
        return tuple(int(x) for x in out)

    def layout(self) -> PagedLayoutC:
        L = PagedLayoutC()
        check(self.L.tkv_pages_layout(self.pages, ct.byref(L)))
        return L

    def device_table(self, qid: int):
        ptr = ct.c_void_p()
        stride = ct.c_uint32(0)
        check(self.L.tkv_pages_device_table(self.pages, qid, self.stream_handle, ct.byref(ptr), ct.byref(stride)))
        return ptr.value, stride.value


def _codec_launch(fn, srcs, dsts, sizes, with_scratch: bool, stream=None):
    from ._lib import CodecItemC
    items = (CodecItemC * len(srcs))(*[CodecItemC(s.data_ptr(), d.data_ptr(), n) for s, d, n in zip(srcs, dsts, sizes)])
    seg = np.zeros(len(srcs) + 1, np.uint32)
    check(lib().tkv_codec_plan(ct.cast(items, ct.c_void_p), len(srcs), seg.ctypes.data_as(u32p)))
    dev = srcs[0].device
    d_items = torch.frombuffer(bytearray(bytes(items)), dtype=torch.uint8).to(dev)
    d_seg = torch.from_numpy(seg.view(np.int32)).to(dev)
    s = stream.cuda_stream if stream is not None else torch.cuda.current_stream(dev).cuda_stream
    if with_scratch:
        nbytes = int(lib().tkv_q8_encode_scratch_bytes(len(srcs)))
        scratch = torch.zeros(nbytes // 4, dtype=torch.int32, device=dev)
        check(fn(d_items.data_ptr(), d_seg.data_ptr(), len(srcs), int(seg[-1]), scratch.data_ptr(), s))
    else:
        check(fn(d_items.data_ptr(), d_seg.data_ptr(), len(srcs), int(seg[-1]), s))
    torch.cuda.synchronize(dev)


def q8_encode(payloads: list[torch.Tensor]) -> list[torch.Tensor]:
    """q8-scale blobs of device uint8 payloads, one batched launch (codec.cpp:27-91)."""
    blobs = [torch.empty(int(lib().tkv_q8_blob_bytes(p.numel())), dtype=torch.uint8, device=p.device)
             for p in payloads]
    _codec_launch(lib().tkv_q8_encode, payloads, blobs, [p.numel() for p in payloads], True)
    return blobs


def q8_decode(blobs: list[torch.Tensor], lengths: list[int]) -> list[torch.Tensor]:
    outs = [torch.empty(n, dtype=torch.uint8, device=b.device) for b, n in zip(blobs, lengths)]
    _codec_launch(lib().tkv_q8_decode, blobs, outs, lengths, False)
    return outs


class PdStaging:
    """Decoder landing area (pd_staging.hpp contract) over the C-ABI."""

    def __init__(self):
        self.L = lib()
        self.h = ct.c_void_p()
        check(self.L.tkv_pd_staging_create(ct.byref(self.h)))

    def close(self):
        if self.h:
            self.L.tkv_pd_staging_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def register_query(self, qid: int) -> int:
        return self.L.tkv_pd_register(self.h, qid)

    def push(self, qid: int, ordinal: int, last: bool, rec: PdRecordC | None = None) -> int:
        rec = rec if rec is not None else PdRecordC()
        return self.L.tkv_pd_push(self.h, qid, ordinal, int(last), ct.byref(rec))

    def await_(self, qid: int):
        cap = 1 << 14
        out = (PdRecordC * cap)()
        n = ct.c_size_t(0)
        rc = self.L.tkv_pd_await(self.h, qid, out, cap, ct.byref(n))
        return rc, [out[i] for i in range(n.value)] if rc == 0 else []

    def cancel(self, qid: int) -> int:
        return self.L.tkv_pd_cancel(self.h, qid)

    def registered(self) -> int:
        return int(self.L.tkv_pd_registered(self.h))


def pd_send(engine: "Engine", qid: int, n_tokens: int, landing_ptr: int, chunk_stride: int):
    """Prefiller: gather the query's chunks (all layers) into landing memory."""
    cap = (n_tokens + engine.chunk_size - 1) // engine.chunk_size + 1
    out = (PdRecordC * cap)()
    n = ct.c_size_t(0)
    check(lib().tkv_pd_send(engine.pages, qid, n_tokens, engine.chunk_size, landing_ptr, chunk_stride,
                            engine.stream_handle, out, cap, ct.byref(n)))
    return [out[i] for i in range(n.value)]


def pd_send_staged(engine: "Engine", qid: int, n_tokens: int, landing_ptr: int, chunk_stride: int,
                   staging_ptr: int, group_bytes: int = 0):
    """Prefiller, copy-engine variant: K1 into local staging, CE peer copies."""
    cap = (n_tokens + engine.chunk_size - 1) // engine.chunk_size + 1
    out = (PdRecordC * cap)()
    n = ct.c_size_t(0)
    check(lib().tkv_pd_send_staged(engine.pages, qid, n_tokens, engine.chunk_size, landing_ptr, chunk_stride,
                                   staging_ptr, group_bytes, engine.stream_handle, out, cap, ct.byref(n)))
    return [out[i] for i in range(n.value)]


class PdLayerSender:
    """Layer-streamed PD send (chunk or page granularity): layer(l) after the
    engine computed layer l, finish() -> records, one per unit."""

    def __init__(self, engine: "Engine", qid: int, n_tokens: int, unit_tokens: int, landing_ptr: int,
                 unit_stride: int):
        self.L = lib()
        self.e = engine
        self.h = ct.c_void_p()
        check(self.L.tkv_pd_sender_begin(engine.pages, qid, n_tokens, unit_tokens, landing_ptr, unit_stride,
                                         ct.byref(self.h)))

    def layer(self, layer: int) -> int:
        return self.L.tkv_pd_sender_layer(self.h, layer, self.e.stream_handle)

    def finish(self):
        cap = 1 << 16
        out = (PdRecordC * cap)()
        n = ct.c_size_t(0)
        check(self.L.tkv_pd_sender_finish(self.h, out, cap, ct.byref(n)))
        return [out[i] for i in range(n.value)]

    def close(self):
        if self.h:
            self.L.tkv_pd_sender_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def pd_land(engine: "Engine", qid: int, records) -> None:
    """Decoder: scatter landed chunks into the query's pages (one launch)."""
    arr = (PdRecordC * max(1, len(records)))(*records)
    check(lib().tkv_pd_land(engine.pages, qid, arr, len(records), engine.stream_handle))


def _model_seed(tag: str) -> int:
    """fnv1a64(model_tag) (synth.hpp:27-30): a per-model constant."""
    h = 0xcbf29ce484222325
    for b in tag.encode():
        h ^= b
        h = (h * 0x100000001b3) & 0xFFFFFFFFFFFFFFFF
    return h
