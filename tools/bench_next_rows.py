"""Measurements for the SURVEY.md §8(f) rows beyond the memo and the codec
(which have tools/bench_lookup.py and tools/bench_codec.py), with the
reference (oracle/_ref) timed beside each on the same inputs:

  decode  delayed decode storing (store.cpp:964-1039, connector.cpp:434-497):
          8B KV, a 4096-token prompt prefilled, then 2048 generated tokens
          appended one at a time (the engine computes each token's KV first);
          every completed 256-token chunk is flushed to the pinned tier.
          Reports the host latency of append_decode per token (finish_query
          included), the engine's per-token compute excluded on both sides.
          The B200 flush is asynchronous (K1 into the pinned slot on the store
          stream, committed by a stream callback), so it overlaps the engine's
          next tokens; the reference copies the chunk on the calling thread.
  record  LMCK record framing (chunk_file.cpp:7-95): export of one 8B chunk
          (32 MiB payload) from the tier as a record and import back,
          GB/s of payload, against the reference's encode/parse.
One JSON line per row."""
import ctypes as ct
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import oracle  # noqa: E402
from paper_2510_09665_b200._lib import u8p  # noqa: E402
from paper_2510_09665_b200.api import Engine  # noqa: E402

TAG, L, BPT = "llama-3.1-8b", 32, 4096


def toks(n, seed):
    return np.random.default_rng(seed).integers(0, 128256, size=n, dtype=np.uint32)


def decode_run(factory, prompt, gen):
    """Prefill `prompt`, then append `gen`; returns (append seconds, flushed keys)."""
    n_all = len(prompt) + len(gen)
    e = factory(num_layers=L, bpt=BPT, page_tokens=16, tag=TAG, chunk_size=256, ram_slots=64,
                num_pages=(n_all // 16 + 16) * L)
    q = 1
    e.get_num_new_matched_tokens(q, prompt)
    e.bind_pages(q, n_all)
    e.update_state_after_alloc(q, (n_all + 15) // 16, 0)
    m = e.build_connector_meta([(q, prompt)])
    full = np.concatenate([prompt, gen]).astype(np.uint32)
    e.start_load_kv(m)
    if hasattr(e, "stream_handle"):
        for layer in range(L):
            e.wait_load_kv(m, layer)
            e.compute_range(q, full, 0, len(prompt), layers=(layer, layer + 1))
            if layer:
                e.wait_store_kv(m, layer - 1)
            e.start_store_kv(m)
    else:
        e.compute_range(q, full, 0, len(prompt))
        for layer in range(L):
            e.wait_load_kv(m, layer)
            if layer:
                e.wait_store_kv(m, layer - 1)
            e.start_store_kv(m)
    e.wait_store_kv(m, L - 1)
    assert e.begin_decode(q) == 0
    t = 0.0
    for i, tok in enumerate(gen):
        e.compute_range(q, full, len(prompt) + i, len(prompt) + i + 1)  # the engine's compute (untimed)
        if hasattr(e, "synchronize"):
            e.synchronize()
        t0 = time.perf_counter()
        assert e.append_decode(q, int(tok)) == 0
        t += time.perf_counter() - t0
    t0 = time.perf_counter()
    keys, rc = e.finish_query_keys(q)
    t += time.perf_counter() - t0
    assert rc == 0
    e.close()
    return t, keys


def bench_decode():
    prompt, gen = toks(4096, 1), toks(2048, 2)
    t_gpu, k_gpu = decode_run(Engine, prompt, gen)
    out = {"row": "decode storing", "prompt": len(prompt), "generated": len(gen),
           "flushed_chunks": len(k_gpu), "append_us_per_token": round(1e6 * t_gpu / len(gen), 2)}
    if oracle.ref_available():
        t_ref, k_ref = decode_run(oracle.RefEngine, prompt, gen)
        out.update({"keys_equal_reference": k_gpu == k_ref,
                    "ref_append_us_per_token": round(1e6 * t_ref / len(gen), 2)})
    return out


def bench_record(reps=5):
    C = oracle.C()
    prompt = toks(256, 3)
    e = Engine(num_layers=L, bpt=BPT, page_tokens=16, tag=TAG, chunk_size=256, ram_slots=4, num_pages=64)
    e.seed_store(prompt, 256)
    key = C.chunk_keys(prompt, 256, TAG)[0]
    lib = e.L
    th = ct.c_uint64(0)
    assert lib.tkv_model_tag_hash(TAG.encode(), ct.byref(th)) == 0
    d = np.frombuffer(key, np.uint8).copy()
    n = ct.c_size_t(0)
    lib.tkv_store_export_record(e.store, d.ctypes.data_as(u8p), th.value, None, 0, ct.byref(n))
    rec = np.zeros(n.value, np.uint8)
    te, ti = [], []
    for _ in range(reps):
        t0 = time.perf_counter()
        assert lib.tkv_store_export_record(e.store, d.ctypes.data_as(u8p), th.value, rec.ctypes.data_as(u8p),
                                           rec.size, ct.byref(n)) == 0
        te.append(time.perf_counter() - t0)
    f = Engine(num_layers=L, bpt=BPT, page_tokens=16, tag=TAG, chunk_size=256, ram_slots=reps + 1, num_pages=64)
    for _ in range(reps):
        assert f.store_clear(key) in (0, 1)
        t0 = time.perf_counter()
        assert lib.tkv_store_import_record(f.store, rec.ctypes.data_as(u8p), rec.size, 0) == 0
        ti.append(time.perf_counter() - t0)
    payload = 256 * L * BPT
    out = {"row": "LMCK record framing", "payload_bytes": payload,
           "export_gbps": round(payload / min(te) / 1e9, 3), "import_gbps": round(payload / min(ti) / 1e9, 3)}
    if oracle.ref_available():
        R = oracle.Ref()
        pay = C.synth_chunk(C.model_seed(TAG), prompt, 0, 256, L, BPT)
        t0 = time.perf_counter()
        want = R.encode_record(TAG, key, 256, L, BPT, pay)
        t1 = time.perf_counter()
        code, _ = R.parse_record(want, pay.size)
        t2 = time.perf_counter()
        out.update({"bytes_equal_reference": bool(np.array_equal(rec, want)) and code == 0,
                    "ref_encode_gbps": round(payload / (t1 - t0) / 1e9, 3),
                    "ref_parse_gbps": round(payload / (t2 - t1) / 1e9, 3)})
    e.close()
    f.close()
    return out


if __name__ == "__main__":
    torch.cuda.init()
    print(json.dumps(bench_decode()), flush=True)
    print(json.dumps(bench_record()), flush=True)
