"""BASELINE.json configs 1, 2 and 4 through the C-ABI connector (bench.py's
`configs` object; also runnable alone, one JSON line per config).

  c1  8B KV (32 L x 4096 B), one 4K-token prompt: cold store, then warm
      retrieve (len-1 tokens), chunk 256, page 16.
  c2  8B KV, 64 requests, lengths seeded uniform over multiples of 256 in
      [8192, 32768]; prefix-hit retrieve from the pinned tier, the requests of
      a wave in ONE scheduling iteration (batched lookup, one metadata,
      layerwise). All 64 run; 160 GiB of KV does not fit the host tier at
      once, so they go in waves (each wave stored untimed, then retrieved
      timed); stated in the line.
  c4  8B KV, multi-round QA: 3 shared 131,072-token documents + a 20-100
      token question per query; seeded 50 % / 90 % document reuse; lookup
      (K3 + LPM) + retrieve of the document prefix (hits) or cold store
      (misses). Lookup latency split by hit / miss.
  c5  PD transfer. Across GPUs (NVLink pairs) only at N >= 2: bench.py's
      "pd". Here c5_loopback: the same pair transfer (70B KV, TP=4 head
      shard, 32K tokens = 2.5 GiB) with prefill and decode engines on ONE
      GPU — every send path, the PdStaging ordinal contract and the land,
      byte-verified; HBM-bound, not an NVLink number.

Every config verifies its bytes on the device after the timed work: the page
image of every request against synth (retrieved prefix + computed tokens),
and the tier slots it stored (read over PCIe by the SMs) against synth.
Each carries the reference Connector (oracle/_ref, CPU) on the same inputs
(bounded where it would take minutes; the sample is stated) and the fraction
of the in-run PCIe rates (one way for one-directional configs).
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

from paper_2510_09665_b200.api import Engine, chunk_keys  # noqa: E402

TAG8 = "llama-3.1-8b"
L8, BPT8 = 32, 4096


def toks(n, seed, vocab=128256):
    return np.random.default_rng(seed).integers(0, vocab, size=n, dtype=np.uint32)


class Verifier:
    """Device byte checks accumulated over a config run."""

    def __init__(self):
        self.page_words = 0   # mismatching 8-byte words in page images
        self.pages_checked = 0
        self.slot_words = 0   # mismatching words in stored tier slots
        self.slots_checked = 0

    def pages(self, e, q, p):
        self.page_words += e.verify_range(q, p, 0, len(p))
        self.pages_checked += 1

    def slots(self, e, p, first_chunk=0):
        keys = chunk_keys(p, 256, e.tag)
        for i in range(first_chunk, len(keys)):
            r = e.verify_stored(keys[i], p, 256 * i)
            if r is not None:
                self.slot_words += r
                self.slots_checked += 1

    def out(self):
        return {"page_mismatch_words": self.page_words, "requests_checked": self.pages_checked,
                "slot_mismatch_words": self.slot_words, "slots_checked": self.slots_checked}


def run_batch(e, queries, matched=None, verify=None):
    """One scheduling iteration for [(qid, prompt)] with the reference call
    order; returns (loaded tokens, stored tokens). `matched`: the lookup was
    already done by the scheduler. `verify` (a Verifier) checks every page
    image before the pages are released (outside any timing the caller does
    only if the caller stops its clock first; configs verify after timing)."""
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
    return sum(loaded.values()), stored


def finish(e, queries, verify=None):
    for q, p in queries:
        if verify is not None:
            verify.pages(e, q, p)
        e.finish_query(q)
        e.release_query(q)


def ref_batch_gbps(queries, L, bpt, tag, stored_prefix):
    """Reference Connector (CPU) on the same batch shape; connector calls only
    (lookup, alloc update, meta, loads, stores), engine compute excluded."""
    import oracle
    if not oracle.ref_available():
        return None
    threads = len(os.sched_getaffinity(0))
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
    return {"value": round((loaded + stored) * L * bpt / t / 1e9, 4), "unit": "GB/s", "seconds": round(t, 3),
            "cores": threads, "kind": "reference", "lookup_ms": round(1e3 * t_lookup, 3)}


def _fracs(gbps, pcie, both=False):
    if not pcie:
        return {}
    one = min(pcie["h2d_gbps"], pcie["d2h_gbps"])
    out = {"frac_of_pcie_one_way": round(gbps / one, 4)}
    if both:
        out["frac_of_pcie_bidir"] = round(gbps / pcie["bidir_gbps"], 4)
    return out


def c1(reps=3, pcie=None, cpu=True):
    """Config 1: one 4K-token prompt, cold store then warm retrieve."""
    n = 4096
    e = Engine(num_layers=L8, bpt=BPT8, page_tokens=16, tag=TAG8, chunk_size=256, ram_slots=4 * 17 + 8,
               num_pages=2 * (n // 16 + 16) * L8, staging_budget=1 << 34, stream=torch.cuda.Stream())
    v = Verifier()
    st, rt = [], []
    qid = 1
    for r in range(reps + 1):
        p = toks(n, 100 + r)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        lo, so = run_batch(e, [(qid, p)])
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        finish(e, [(qid, p)], v)
        v.slots(e, p)
        torch.cuda.synchronize()
        t1b = time.perf_counter()
        lo2, so2 = run_batch(e, [(qid + 1, p)])
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        finish(e, [(qid + 1, p)], v)
        qid += 2
        assert lo == 0 and so == n and lo2 == n - 1 and so2 == 0
        if r:
            st.append(t1 - t0)
            rt.append(t2 - t1b)
    sb, rb = n * L8 * BPT8, (n - 1) * L8 * BPT8
    s, r_ = float(np.median(st)), float(np.median(rt))
    host_copies = dict(zip(("host_tier_pieces", "host_tier_copies"), e.copy_runs()))
    e.close()
    out = {"workload": "c1: Llama-3.1-8B KV (32 L x 4096 B), one 4096-token prompt: cold store, then warm "
                       "retrieve (4095 tokens), chunk 256, page 16",
           "store_gbps": round(sb / s / 1e9, 2), "store_ms": round(1e3 * s, 3),
           "retrieve_gbps": round(rb / r_ / 1e9, 2), "retrieve_ms": round(1e3 * r_, 3),
           "e2e": {"value": round((sb + rb) / (s + r_) / 1e9, 2), "unit": "GB/s",
                   "tokens_per_s": round((2 * n - 1) / (s + r_), 1), "reps": reps},
           "store": _fracs(sb / s / 1e9, pcie), "retrieve": _fracs(rb / r_ / 1e9, pcie),
           "verify": v.out(), **host_copies}
    if cpu:
        ref_s = ref_batch_gbps([(1, toks(n, 100))], L8, BPT8, TAG8, lambda p: 0)
        ref_r = ref_batch_gbps([(1, toks(n, 100))], L8, BPT8, TAG8, lambda p: len(p))
        if ref_s and ref_r:
            t = sb / (ref_s["value"] * 1e9) + rb / (ref_r["value"] * 1e9)
            out["cpu_baseline"] = {"value": round((sb + rb) / t / 1e9, 4), "unit": "GB/s", "kind": "reference",
                                   "cores": ref_s["cores"], "store_gbps": ref_s["value"],
                                   "retrieve_gbps": ref_r["value"],
                                   "sample": "the same prompt: one cold store + one warm retrieve (full config)"}
    return out


def c2(wave=8, pcie=None, cpu=True, n_req=64):
    """Config 2: 64 requests 8K-32K, prefix-hit retrieve, waves of `wave`."""
    rng = np.random.default_rng(64)
    lens = (rng.integers(8192 // 256, 32768 // 256 + 1, size=n_req) * 256).tolist()
    max_wave_tokens = sum(sorted(lens)[-wave:])
    e = Engine(num_layers=L8, bpt=BPT8, page_tokens=16, tag=TAG8, chunk_size=256,
               ram_slots=max_wave_tokens // 256 + wave + 8,
               num_pages=(max_wave_tokens // 16 + 16 * wave) * L8 + (32768 // 16 + 16) * L8,
               staging_budget=1 << 36, stream=torch.cuda.Stream())
    v = Verifier()
    total_loaded, total_t, waves = 0, 0.0, []
    qid = 1000
    for w0 in range(0, n_req, wave):
        batch = [(qid + i, toks(n, 5000 + w0 + i)) for i, n in enumerate(lens[w0:w0 + wave])]
        qid += wave
        for q, p in batch:  # pre-store (untimed): one cold prefill per request
            run_batch(e, [(q + 100000, p)])
            finish(e, [(q + 100000, p)])
        for q, p in batch:  # the stored slots, checked before they are retrieved
            v.slots(e, p)
        if w0 == 0:  # warm-up (untimed): the first retrieve grows rings and plan pools
            warm = [(q + 200000, p) for q, p in batch]
            run_batch(e, warm)
            finish(e, warm)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        lo, so = run_batch(e, batch)
        torch.cuda.synchronize()
        t = time.perf_counter() - t0
        finish(e, batch, v)
        assert so == 0 and lo == sum(len(p) - 1 for _, p in batch)
        total_loaded += lo
        total_t += t
        waves.append(round(lo * L8 * BPT8 / t / 1e9, 2))
    gb = total_loaded * L8 * BPT8
    host_copies = dict(zip(("host_tier_pieces", "host_tier_copies"), e.copy_runs()))
    e.close()
    out = {"workload": f"c2: Llama-3.1-8B KV, {n_req} requests of 8K-32K tokens (mean {int(np.mean(lens))}), "
                       f"prefix-hit retrieve from the pinned tier, {wave} requests per scheduling iteration "
                       f"({n_req // wave} waves; each wave stored untimed, then retrieved timed; one untimed "
                       f"warm-up retrieve of the first wave)",
           "e2e": {"value": round(gb / total_t / 1e9, 2), "unit": "GB/s",
                   "tokens_per_s": round(total_loaded / total_t, 1), "bytes": gb, "seconds": round(total_t, 3)},
           "wave_gbps": waves, **_fracs(gb / total_t / 1e9, pcie), "verify": v.out(), **host_copies}
    if cpu:
        sample = batch[:1]
        ref = ref_batch_gbps(sample, L8, BPT8, TAG8, lambda p: len(p))
        if ref:
            out["cpu_baseline"] = {**ref, "sample": f"one {len(sample[0][1])}-token request of the last wave "
                                                    f"(prefix-hit retrieve, all 32 layers)"}
    return out


def c4(queries=8, reuse=0.5, pcie=None, cpu=True):
    """Config 4: multi-round QA over 128K shared documents."""
    n_doc, n_docs = 131072, 3
    rng = np.random.default_rng(int(reuse * 100))
    docs = [toks(n_doc, 7000 + d) for d in range(n_docs)]
    e = Engine(num_layers=L8, bpt=BPT8, page_tokens=16, tag=TAG8, chunk_size=256,
               ram_slots=(n_docs + 1) * (n_doc // 256 + 1), num_pages=(n_doc // 16 + 64) * L8 + 64,
               staging_budget=1 << 36, stream=torch.cuda.Stream())
    v = Verifier()
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
        torch.cuda.synchronize()
        t_total += time.perf_counter() - t0
        finish(e, [(qid, prompt)], v)
        moved += (lo + so) * L8 * BPT8
        hits += d in seen
        misses += d not in seen
        hit_flags.append(d in seen)
        seen.add(d)
        qid += 1
    for d in sorted(seen):  # every stored document chunk still in the tier
        v.slots(e, docs[d])
    # The lookups measured the way the reference's are below: best of 3 on one
    # prompt, query state dropped between (the in-loop numbers above are one
    # first-time lookup per query, in the middle of the transfers).
    probe = {}
    stored = sorted(seen)[0]
    for kind, p in (("hit", np.concatenate([docs[stored], toks(60, 1)])), ("miss", toks(n_doc, 7777))):
        best = 1e9
        for _ in range(3):
            e.dev_prompt(qid, p)  # the engine's own prompt upload, as in the loop above
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            e.get_num_new_matched_tokens(qid, p)
            best = min(best, time.perf_counter() - t0)
            e.finish_query(qid)
        probe[kind] = round(1e3 * best, 3)
        qid += 1
    memo = e.memo_stats()
    host_copies = dict(zip(("host_tier_pieces", "host_tier_copies"), e.copy_runs()))
    e.close()
    med = (lambda xs: round(1e3 * float(np.median(xs)), 3) if xs else None)
    out = {"workload": f"c4: Llama-3.1-8B KV, {n_docs} shared 131072-token documents + 20-100 token question, "
                       f"document reuse {reuse:.0%}, {queries} queries (lookup + retrieve, or cold store)",
           "hits": hits, "misses": misses,
           "e2e": {"value": round(moved / t_total / 1e9, 2), "unit": "GB/s",
                   "tokens_per_s": round(moved / (L8 * BPT8) / t_total, 1)},
           **_fracs(moved / t_total / 1e9, pcie),
           "lookup_ms_hit": med([t for t, h in zip(t_lookup, hit_flags) if h]),
           "lookup_ms_miss": med([t for t, h in zip(t_lookup, hit_flags) if not h]),
           "lookup_probe_ms": {**probe, "method": "best of 3 on one prompt (a stored document + 60-token "
                                                  "question / a cold 128K document), as the reference's"},
           "memo": memo, "verify": v.out(), **host_copies}
    if cpu:
        import oracle
        if oracle.ref_available():
            # The reference Connector's own lookup on the same prompts (it hashes
            # up to the first absent chunk); the lookup does not depend on the KV
            # geometry, so the reference stack holds the document in 64-byte rows.
            r = oracle.RefEngine(num_layers=1, bpt=64, page_tokens=16, tag=TAG8, chunk_size=256,
                                 ram_slots=n_doc // 256 + 8, num_pages=64)
            r.seed_store(docs[0], n_doc)
            ref_lookup = {}
            for kind, p in (("hit", np.concatenate([docs[0], toks(60, 1)])), ("miss", docs[1])):
                best = 1e9
                for _ in range(3):
                    t0 = time.perf_counter()
                    r.get_num_new_matched_tokens(1, p)
                    best = min(best, time.perf_counter() - t0)
                    r.finish_query(1)
                ref_lookup[kind] = round(1e3 * best, 3)
            r.close()
            sample = [(1, np.concatenate([docs[0], toks(60, 1)]))]
            ref = ref_batch_gbps(sample, 4, BPT8, TAG8, lambda p: n_doc)
            out["cpu_baseline"] = {**(ref or {}), "lookup_ms_hit": ref_lookup["hit"],
                                   "lookup_ms_miss": ref_lookup["miss"],
                                   "sample": "transfer: one document hit + question, 4 of 32 layers; lookups: "
                                             "the reference Connector's own lookup of a stored / cold document"}
    return out


def c5_loopback(reps=3, cpu=True, n=32768, L=80):
    """Config 5's per-pair PD transfer (run_pd, src/sim_engine.cpp:374-472)
    with the prefill and the decode engine on the same GPU: the prefilled
    32K-token prompt's KV (70B, 80 layers, TP=4 head shard: bpt 1024) moves
    into the decoder's landing buffer by each send path — K1 straight into
    the landing buffer (SM-direct), K1 into local staging + copy-engine copy
    (CE-staged), and layer-streamed at page (16-token window) granularity —
    then the decoder takes the chunk records out of order with a duplicate
    through PdStaging, lands them with one K2 and checks every page word
    against synth. Same device, so the bound is HBM (K1 reads and writes each
    byte: 2 x payload), not NVLink."""
    from paper_2510_09665_b200.api import PdLayerSender, PdRecordC, PdStaging, pd_land, pd_send, pd_send_staged
    tag, bpt, q = "llama-3.1-70b", 4096 // 4, 7
    chunks, stride = (n + 255) // 256, L * 256 * bpt
    mk = dict(num_layers=L, bpt=bpt, page_tokens=16, tag=tag, chunk_size=256, ram_slots=2,
              num_pages=(n // 16 + 16) * L, device=0)
    pre, dec = Engine(**mk), Engine(**mk)
    out = {"workload": f"c5 (one GPU): 70B KV ({L} layers), TP=4 shard (bpt 1024), {n}-token prompt, one prefill "
                       f"-> decode pair's chunks ({n * L * bpt / 2**30:.2f} GiB), prefill and decode engines on the "
                       "same B200",
           "note": "no NVLink on a 1-GPU box: the NVLink pairs are bench.py's 'pd' at N >= 2"}
    try:
        prompt = toks(n, 999)
        assert pre.bind_pages(q, n) == 0
        pre.compute_range(q, prompt, 0, n)
        landing = torch.empty(chunks * stride, dtype=torch.uint8, device="cuda")
        staging = torch.empty(chunks * stride, dtype=torch.uint8, device="cuda")
        payload = n * L * bpt
        torch.cuda.synchronize()

        def timed(fn):
            best, res = 1e9, None
            for it in range(reps + 1):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                res = fn()
                torch.cuda.synchronize()
                if it:
                    best = min(best, time.perf_counter() - t0)
            return best, res

        def streamed():
            snd = PdLayerSender(pre, q, n, 16, landing.data_ptr(), L * 16 * bpt)
            for layer in range(L):
                assert snd.layer(layer) == 0
            r = snd.finish()
            snd.close()
            return r
        t_ce, _ = timed(lambda: pd_send_staged(pre, q, n, landing.data_ptr(), stride, staging.data_ptr()))
        t_pg, wrecs = timed(streamed)
        assert len(wrecs) == (n + 15) // 16
        t_sm, recs = timed(lambda: pd_send(pre, q, n, landing.data_ptr(), stride))  # landed bytes come from it
        st = PdStaging()
        assert st.register_query(q) == 0
        for o in list(range(chunks))[::-1] + [0]:  # out of order + a duplicate
            r = recs[o]
            assert st.push(q, o, o == chunks - 1, PdRecordC(addr=r.addr, bytes=r.bytes, token_count=r.token_count,
                                                            first_token=r.first_token)) == 0
        rc, landed = st.await_(q)
        assert rc == 0 and len(landed) == chunks
        assert dec.bind_pages(q, n) == 0
        t_land, _ = timed(lambda: pd_land(dec, q, landed))  # idempotent: the same records each time
        mism = dec.verify_range(q, prompt, 0, n)
        st.close()
        g = lambda t: round(payload / t / 1e9, 1)  # noqa: E731
        out.update({"bytes": payload, "sm_direct_gbps": g(t_sm), "ce_staged_gbps": g(t_ce),
                    "layer_streamed_page_gbps": g(t_pg), "land_gbps": g(t_land),
                    "sm_direct_hbm_algorithmic_gbps": round(2 * payload / t_sm / 1e9, 1),
                    "verify": {"page_mismatch_words": mism, "chunks_landed": len(landed)},
                    "timing": "min of 3 synchronised calls after one warm-up (each send returns after its "
                              "bytes landed)"})
        if cpu:
            sys.path.insert(0, ROOT)
            import bench as _bench
            out["cpu_baseline"] = _bench.reference_pd_gbps(L, bpt)
    finally:
        pre.close()
        dec.close()
    return out


def run_all(pcie=None, cpu=True, wave=8, queries=8):
    out = {}
    for name, fn in (("c1", lambda: c1(3, pcie, cpu)), ("c2", lambda: c2(wave, pcie, cpu)),
                     ("c4_reuse50", lambda: c4(queries, 0.5, pcie, cpu)),
                     ("c4_reuse90", lambda: c4(queries, 0.9, pcie, cpu)),
                     ("c5_loopback", lambda: c5_loopback(3, cpu))):
        t0 = time.time()
        try:
            out[name] = fn()
        except Exception as ex:  # a failing config is reported, not hidden
            out[name] = {"ok": False, "error": repr(ex)[:300]}
        out[name]["wall_s"] = round(time.time() - t0, 1)
        torch.cuda.empty_cache()
    return out


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="c1,c2,c4,c5")
    ap.add_argument("--wave", type=int, default=8)
    ap.add_argument("--queries", type=int, default=8)
    ap.add_argument("--no-cpu", action="store_true")
    a = ap.parse_args()
    cpu = not a.no_cpu
    if "c1" in a.only:
        print(json.dumps(c1(3, cpu=cpu)), flush=True)
    if "c2" in a.only:
        print(json.dumps(c2(a.wave, cpu=cpu)), flush=True)
    if "c4" in a.only:
        print(json.dumps(c4(a.queries, 0.5, cpu=cpu)), flush=True)
        print(json.dumps(c4(a.queries, 0.9, cpu=cpu)), flush=True)
    if "c5" in a.only:
        print(json.dumps(c5_loopback(3, cpu=cpu)), flush=True)
