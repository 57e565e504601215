"""Secondary measurements for the other BASELINE.json configs (one JSON line
each). The driver's headline is bench.py (config 3); these complete
SURVEY.md §8(d)'s "payload GB/s and tokens/s for each config".

  c1  8B KV (32 L x 4096 B), one 4K-token prompt: cold store, then warm
      retrieve (len-1 tokens), chunk 256, page 16.
  c2  8B KV, 64 requests, lengths seeded uniform over multiples of 256 in
      [8192, 32768]; prefix-hit retrieve from the pinned tier, all requests of
      a wave in ONE scheduling iteration (batched lookup, one metadata,
      layerwise). 160 GiB does not fit the 196 GB host at once, so the 64
      requests run in waves (stored untimed, retrieved timed); stated.
  c4  8B KV, multi-round QA: 4 shared 131,072-token documents + a 20-100
      token question per query; seeded 50 % / 90 % document reuse; lookup
      (K3 + LPM) + retrieve of the document prefix (hits) or cold store
      (misses). Reports lookup latency and transfer GB/s.
  c5  needs >= 2 GPUs: bench.py at N >= 2 reports it ("pd").

Each line carries the reference CPU path (oracle/_ref Connector) on a
bounded sample of the same workload where it finishes in seconds.
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2510_09665_b200.api import Engine  # noqa: E402

TAG8 = "llama-3.1-8b"
L8, BPT8 = 32, 4096


def toks(n, seed, vocab=128256):
    return np.random.default_rng(seed).integers(0, vocab, size=n, dtype=np.uint32)


def run_batch(e, queries, matched=None):
    """One scheduling iteration for [(qid, prompt)] with the reference call
    order; returns (loaded tokens, stored tokens). `matched`: the lookup was
    already done by the scheduler."""
    ids = [q for q, _ in queries]
    if matched is None:
        matched = e.lookup_batch(ids, [p for _, p in queries])
    for (q, p), mt in zip(queries, matched):
        assert e.bind_pages(q, len(p)) == 0
        assert e.update_state_after_alloc(q, (len(p) + 15) // 16, (mt + 15) // 16) == 0
    m = e.build_connector_meta(queries)
    assert e.start_load_kv(m) == 0
    loaded = {q: e.loaded_tokens(m, q) for q in ids}
    for layer in range(e.num_layers):
        e.wait_load_kv(m, layer)
        for q, p in queries:
            e.compute_range(q, p, loaded[q], len(p), layers=(layer, layer + 1))
        if layer:
            e.wait_store_kv(m, layer - 1)
        assert e.start_store_kv(m) == 0
    assert e.wait_store_kv(m, e.num_layers - 1) == 0
    stored = 0
    for i, (q, p) in enumerate(queries):
        sp, _ = e.plan(m, i, "store")
        stored += sum(b - a for a, b, _, _, _ in sp)
        assert all(c == 0 for _, c in e.store_results(m, q))
    e.drop_meta(m)
    for q in ids:
        e.finish_query(q)
        e.release_query(q)
    return sum(loaded.values()), stored


def ref_batch_gbps(queries, L, bpt, tag, stored_prefix):
    """Reference Connector (CPU) on the same batch shape; connector calls only."""
    import oracle
    if not oracle.ref_available():
        return None
    threads = os.cpu_count() or 1
    tot = sum(len(p) for _, p in queries)
    e = oracle.RefEngine(num_layers=L, bpt=bpt, page_tokens=16, tag=tag, chunk_size=256,
                         ram_slots=2 * (tot // 256 + len(queries)) + 8,
                         num_pages=2 * (tot // 16 + 16 * len(queries)) * L, layerwise=True,
                         staging_budget=1 << 40, io_threads=threads, store_io_threads=threads)
    for q, p in queries:
        if stored_prefix(p):
            e.seed_store(p, stored_prefix(p))
    for q, p in queries:
        e.bind_pages(q, len(p))
    t0 = time.perf_counter()
    matched = [e.get_num_new_matched_tokens(q, p) for q, p in queries]
    for (q, p), mt in zip(queries, matched):
        e.update_state_after_alloc(q, (len(p) + 15) // 16, (mt + 15) // 16)
    t_lookup = time.perf_counter() - t0
    for (q, p), mt in zip(queries, matched):
        e.compute_range(q, p, mt, len(p))  # engine compute, excluded from the timing
    t1 = time.perf_counter()
    m = e.build_connector_meta(queries)
    e.start_load_kv(m)
    for layer in range(L):
        e.wait_load_kv(m, layer)
        if layer:
            e.wait_store_kv(m, layer - 1)
        e.start_store_kv(m)
    e.wait_store_kv(m, L - 1)
    t = t_lookup + time.perf_counter() - t1
    loaded = sum(e.loaded_tokens(m, q) for q, _ in queries)
    stored = sum(len(p) - mt for (q, p), mt in zip(queries, matched))
    e.close()
    return {"gbps": (loaded + stored) * L * bpt / t / 1e9, "seconds": round(t, 3), "cores": threads,
            "lookup_ms": round(1e3 * t_lookup, 3)}


def c1(reps):
    n = 4096
    e = Engine(num_layers=L8, bpt=BPT8, page_tokens=16, tag=TAG8, chunk_size=256, ram_slots=4 * 17 + 8,
               num_pages=2 * (n // 16 + 16) * L8, staging_budget=1 << 34, stream=torch.cuda.Stream())
    st, rt = [], []
    qid = 1
    for r in range(reps + 1):
        p = toks(n, 100 + r)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        lo, so = run_batch(e, [(qid, p)])
        t1 = time.perf_counter()
        lo2, so2 = run_batch(e, [(qid + 1, p)])
        t2 = time.perf_counter()
        qid += 2
        assert lo == 0 and so == n and lo2 == n - 1 and so2 == 0
        if r:
            st.append(t1 - t0)
            rt.append(t2 - t1)
    sb, rb = n * L8 * BPT8, (n - 1) * L8 * BPT8
    s, r_ = min(st), min(rt)
    ref = ref_batch_gbps([(1, toks(n, 100))], L8, BPT8, TAG8, lambda p: 0)
    ref_w = ref_batch_gbps([(1, toks(n, 100))], L8, BPT8, TAG8, lambda p: len(p))
    e.close()
    return {"config": "c1: 8B KV, 4K prompt, store then retrieve", "store_gbps": round(sb / s / 1e9, 2),
            "store_ms": round(1e3 * s, 3), "retrieve_gbps": round(rb / r_ / 1e9, 2), "retrieve_ms": round(1e3 * r_, 3),
            "store_retrieve_gbps": round((sb + rb) / (s + r_) / 1e9, 2),
            "tokens_per_s": round((2 * n - 1) / (s + r_), 1),
            "ref_cpu": {"store": ref, "retrieve": ref_w}}


def c2(wave):
    rng = np.random.default_rng(64)
    lens = (rng.integers(8192 // 256, 32768 // 256 + 1, size=64) * 256).tolist()
    max_wave_tokens = sum(sorted(lens)[-wave:])
    e = Engine(num_layers=L8, bpt=BPT8, page_tokens=16, tag=TAG8, chunk_size=256,
               ram_slots=max_wave_tokens // 256 + wave + 8,
               num_pages=(max_wave_tokens // 16 + 16 * wave) * L8 + (32768 // 16 + 16) * L8,
               staging_budget=1 << 36, stream=torch.cuda.Stream())
    total_loaded, total_t, lookups = 0, 0.0, []
    qid = 1000
    for w0 in range(0, 64, wave):
        batch = [(qid + i, toks(n, 5000 + w0 + i)) for i, n in enumerate(lens[w0:w0 + wave])]
        qid += wave
        for q, p in batch:  # pre-store (untimed): one cold prefill per request
            run_batch(e, [(q + 100000, p)])
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        lo, so = run_batch(e, batch)
        t = time.perf_counter() - t0
        assert so == 0 and lo == sum(len(p) - 1 for _, p in batch)
        total_loaded += lo
        total_t += t
        if os.environ.get("TKV_C2_WAVES"):
            print(json.dumps({"wave": w0 // wave, "gbps": round(lo * L8 * BPT8 / t / 1e9, 2), "s": round(t, 3)}),
                  file=sys.stderr, flush=True)
    gb = total_loaded * L8 * BPT8
    small = [(1, toks(lens[0], 5000))]
    ref = ref_batch_gbps(small, 8, BPT8, TAG8, lambda p: len(p))
    e.close()
    return {"config": f"c2: 8B KV, 64 requests 8K-32K (mean {int(np.mean(lens))}), prefix-hit retrieve, "
                      f"waves of {wave} requests per scheduling iteration",
            "retrieve_gbps": round(gb / total_t / 1e9, 2), "seconds": round(total_t, 3),
            "tokens_per_s": round(total_loaded / total_t, 1), "bytes": gb,
            "ref_cpu": {"sample": f"one {lens[0]}-token request, 8 of 32 layers", **(ref or {})}}


def c4(queries, reuse):
    n_doc, n_docs = 131072, 3
    rng = np.random.default_rng(int(reuse * 100))
    docs = [toks(n_doc, 7000 + d) for d in range(n_docs)]
    e = Engine(num_layers=L8, bpt=BPT8, page_tokens=16, tag=TAG8, chunk_size=256,
               ram_slots=(n_docs + 1) * (n_doc // 256 + 1), num_pages=(n_doc // 16 + 64) * L8 + 64,
               staging_budget=1 << 36, stream=torch.cuda.Stream())
    seen = set()
    hits = misses = 0
    hit_flags = []
    t_lookup, t_total, moved, qid = [], 0.0, 0, 1
    for i in range(queries):
        if seen and rng.random() < reuse:
            d = int(rng.choice(sorted(seen)))
        else:
            d = next((x for x in range(n_docs) if x not in seen), int(rng.integers(0, n_docs)))
        q_tokens = toks(int(rng.integers(20, 101)), 9000 + i)
        prompt = np.concatenate([docs[d], q_tokens])
        e.dev_prompt(qid, prompt)  # the engine's own prompt upload, not part of the lookup
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        m = e.get_num_new_matched_tokens(qid, prompt)
        t_lookup.append(time.perf_counter() - t0)
        lo, so = run_batch(e, [(qid, prompt)], matched=[m])
        t_total += time.perf_counter() - t0
        moved += (lo + so) * L8 * BPT8
        hits += d in seen
        misses += d not in seen
        hit_flags.append(d in seen)
        seen.add(d)
        qid += 1
    import oracle
    ref_lookup = None
    if oracle.ref_available():
        # The reference Connector's own lookup on the same prompts (hashing up
        # to the first absent chunk); the lookup does not depend on the KV
        # geometry, so the reference stack holds the document in 64-byte rows.
        r = oracle.RefEngine(num_layers=1, bpt=64, page_tokens=16, tag=TAG8, chunk_size=256,
                             ram_slots=n_doc // 256 + 8, num_pages=64)
        r.seed_store(docs[0], n_doc)
        ref_lookup = {}
        for kind, p in (("hit", np.concatenate([docs[0], toks(60, 1)])), ("miss", docs[1])):
            t0 = time.perf_counter()
            r.get_num_new_matched_tokens(1, p)
            ref_lookup[kind] = round(1e3 * (time.perf_counter() - t0), 3)
            r.finish_query(1)
        r.close()
    memo = e.memo_stats()
    e.close()
    return {"config": f"c4: 8B KV, {n_docs} shared 128K docs + question, reuse {reuse:.0%}, {queries} queries",
            "hits": hits, "misses": misses, "gbps": round(moved / t_total / 1e9, 2),
            "lookup_ms_median": round(1e3 * float(np.median(t_lookup)), 3),
            "lookup_ms_hit": round(1e3 * float(np.median([t for t, h in zip(t_lookup, hit_flags) if h] or [0])), 3),
            "lookup_ms_miss": round(1e3 * float(np.median([t for t, h in zip(t_lookup, hit_flags) if not h] or [0])), 3),
            "lookup_tokens_per_s": round((n_doc + 60) / float(np.median(t_lookup)), 1),
            "memo": memo, "ref_cpu_lookup_ms": ref_lookup}


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="c1,c2,c4")
    ap.add_argument("--wave", type=int, default=8)
    ap.add_argument("--queries", type=int, default=8)
    a = ap.parse_args()
    if "c1" in a.only:
        print(json.dumps(c1(3)), flush=True)
    if "c2" in a.only:
        print(json.dumps(c2(a.wave)), flush=True)
    if "c4" in a.only:
        print(json.dumps(c4(a.queries, 0.5)), flush=True)
        print(json.dumps(c4(a.queries, 0.9)), flush=True)
