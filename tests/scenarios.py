"""Engine-agnostic scenarios ported from the reference's connector tests
(tests/test_connector.cpp). Each takes an engine factory — either
``oracle.RefEngine`` (the unmodified reference, CPU) or
``paper_2510_09665_b200.api.Engine`` (this repo, B200) — drives it exactly
like the reference test drives its Connector, and returns a plain dict of
observable outcomes (hit lengths, plans, loaded tokens, page bytes, stored
payloads, statuses). Parity = the two dicts are equal.
"""
from __future__ import annotations

import hashlib

import numpy as np

CONN = dict(num_layers=4, bpt=64, page_tokens=16, tag="conn-test", chunk_size=32)


def ref_factory(**kw):
    """The reference engine as the parity oracle: one store I/O thread and one
    connector I/O thread, so its puts apply in batch_put order. With several
    threads its write_tier tasks race for slots and the LRU victims of an
    overfull batch vary from run to run (observed on a 16-core host); the
    sequential order is the one its code states (store.cpp:500-506)."""
    import oracle
    return oracle.RefEngine(**kw, io_threads=1, store_io_threads=1)


def make_prompt(n: int, seed: int, vocab: int = 32000) -> np.ndarray:
    rng = np.random.default_rng(seed)
    return rng.integers(0, vocab, size=n, dtype=np.uint32)


def run_transfer_ref(e, m, qid, prompt):
    """Reference flavour: compute_range covers all layers (test helper)."""
    n_layers = e.num_layers
    assert e.start_load_kv(m) == 0
    layerwise = e.meta_layerwise(m)
    for layer in range(n_layers):
        if layerwise:
            assert e.wait_load_kv(m, layer) == 0
        loaded = e.loaded_tokens(m, qid)
        e.compute_range(qid, prompt, loaded, len(prompt))
        if layerwise:
            if layer > 0:
                assert e.wait_store_kv(m, layer - 1) == 0
            assert e.start_store_kv(m) == 0
    if layerwise:
        assert e.wait_store_kv(m, n_layers - 1) == 0
    else:
        assert e.start_store_kv(m) == 0


def transfer(e, m, qid, prompt):
    if hasattr(e, "stream_handle"):
        # B200 engine: compute each layer just before its store (engine order).
        n_layers = e.num_layers
        assert e.start_load_kv(m) == 0
        layerwise = e.meta_layerwise(m)
        for layer in range(n_layers):
            if layerwise:
                assert e.wait_load_kv(m, layer) == 0
            loaded = e.loaded_tokens(m, qid)
            e.compute_range(qid, prompt, loaded, len(prompt), layers=(layer, layer + 1))
            if layerwise:
                if layer > 0:
                    assert e.wait_store_kv(m, layer - 1) == 0
                assert e.start_store_kv(m) == 0
        if layerwise:
            assert e.wait_store_kv(m, n_layers - 1) == 0
        else:
            assert e.start_store_kv(m) == 0
    else:
        run_transfer_ref(e, m, qid, prompt)


def page_image(e, qid, n_tokens):
    """sha256 of every layer's gathered bytes for tokens [0, n)."""
    h = hashlib.sha256()
    for layer in range(e.num_layers):
        h.update(e.gather_layer(qid, layer, n_tokens).tobytes())
    return h.hexdigest()


def pages_equal_synth(e, qid, prompt, n_tokens, C):
    seed = C.model_seed(e.tag)
    for layer in range(e.num_layers):
        want = C.synth_layer_kv(seed, prompt[:n_tokens], layer, 0, e.bpt)
        if not np.array_equal(e.gather_layer(qid, layer, n_tokens), want):
            return False
    return True


def plan_view(e, m, qi):
    lp, matched = e.plan(m, qi, "load")
    sp, _ = e.plan(m, qi, "store")
    return {"matched": matched, "load": [(a, b, r, d.hex()) for a, b, r, _, d in lp],
            "store": [(a, b, r, d.hex()) for a, b, r, _, d in sp]}


# ---------------------------------------------------------------- scenarios

def sc_match_cap(factory, C):
    """test_connector.cpp:182-212."""
    out = {}
    prompt = make_prompt(10000, 7)
    for name, n, p in [("9984", 9984, prompt), ("10000", 10000, prompt), ("512", 512, prompt[:512]),
                       ("cold", 0, prompt)]:
        e = factory(num_layers=2, bpt=8, page_tokens=16, tag="match-cap", chunk_size=256, ram_slots=64,
                    num_pages=8)
        if n:
            e.seed_store(p, n)
        out[name] = e.get_num_new_matched_tokens(1, p)
        e.close()
    return out


def sc_load_plan_clip(factory, C):
    """test_connector.cpp:214-242."""
    e = factory(**CONN, ram_slots=16, num_pages=64)
    prompt = make_prompt(70, 11)
    e.seed_store(prompt, 70)
    out = {"match": e.get_num_new_matched_tokens(9, prompt)}
    e.bind_pages(9, 70)
    out["update"] = e.update_state_after_alloc(9, 5, 5)
    m = e.build_connector_meta([(9, prompt)])
    out["plan"] = plan_view(e, m, 0)
    e.release_query(9)
    e.close()
    return out


def sc_inconsistent_alloc(factory, C):
    """test_connector.cpp:244-258."""
    e = factory(**CONN, ram_slots=16, num_pages=64)
    prompt = make_prompt(64, 13)
    e.seed_store(prompt, 64)
    out = {"match": e.get_num_new_matched_tokens(2, prompt),
           "a": e.update_state_after_alloc(2, 4, 3), "b": e.update_state_after_alloc(2, 3, 4),
           "c": e.update_state_after_alloc(99, 4, 4), "d": e.update_state_after_alloc(2, 4, 4)}
    e.close()
    return out


def sc_partial_match(factory, C):
    """test_connector.cpp:260-312: load the stored prefix, store the rest, rerun."""
    e = factory(**CONN, ram_slots=16, num_pages=64)
    prompt = make_prompt(64, 17)
    e.seed_store(prompt, 32)
    out = {"match1": e.get_num_new_matched_tokens(5, prompt)}
    e.bind_pages(5, 64)
    out["upd1"] = e.update_state_after_alloc(5, 4, 2)
    m = e.build_connector_meta([(5, prompt)])
    out["plan1"] = plan_view(e, m, 0)
    transfer(e, m, 5, prompt)
    out["loaded1"] = e.loaded_tokens(m, 5)
    out["pages1_ok"] = pages_equal_synth(e, 5, prompt, 64, C)
    res = e.store_results(m, 5)
    out["results1"] = [(d.hex(), c) for d, c in res]
    stored = e.store_get(res[0][0])
    want = C.synth_chunk(C.model_seed(e.tag), prompt, 32, 32, e.num_layers, e.bpt)
    out["stored_ok"] = stored is not None and np.array_equal(stored, want)
    out["finish1"] = e.finish_query(5)
    e.release_query(5)
    out["match2"] = e.get_num_new_matched_tokens(6, prompt)
    e.bind_pages(6, 64)
    out["upd2"] = e.update_state_after_alloc(6, 4, 4)
    m2 = e.build_connector_meta([(6, prompt)])
    out["plan2"] = plan_view(e, m2, 0)
    transfer(e, m2, 6, prompt)
    out["loaded2"] = e.loaded_tokens(m2, 6)
    out["pages2_ok"] = pages_equal_synth(e, 6, prompt, 64, C)
    out["finish2"] = e.finish_query(6)
    e.release_query(6)
    out["free_all"] = e.free_page_count() == 64
    e.close()
    return out


def sc_layerwise_vs_blocking(factory, C):
    """test_connector.cpp:314-358: same end state in both modes."""
    prompt = make_prompt(96, 23)
    out = {}
    for layerwise in (True, False):
        e = factory(**CONN, ram_slots=16, num_pages=64, layerwise=layerwise)
        e.seed_store(prompt, 64)
        key = "layerwise" if layerwise else "blocking"
        out[key + "_match"] = e.get_num_new_matched_tokens(1, prompt)
        e.bind_pages(1, 96)
        e.update_state_after_alloc(1, 6, 4)
        m = e.build_connector_meta([(1, prompt)])
        transfer(e, m, 1, prompt)
        out[key + "_loaded"] = e.loaded_tokens(m, 1)
        res = e.store_results(m, 1)
        stored = e.store_get(res[0][0])
        out[key + "_image"] = page_image(e, 1, 96) + hashlib.sha256(stored.tobytes()).hexdigest()
        out[key + "_ok"] = pages_equal_synth(e, 1, prompt, 96, C)
        e.finish_query(1)
        e.release_query(1)
        e.close()
    return out


def sc_vanishing_chunk(factory, C):
    """test_connector.cpp:360-385: a chunk cleared after planning shortens
    the delivered prefix; the engine recomputes the tail."""
    e = factory(**CONN, ram_slots=16, num_pages=64)
    prompt = make_prompt(96, 29)
    e.seed_store(prompt, 64)
    keys = C.chunk_keys(prompt[:64], 32, CONN["tag"])
    out = {"match": e.get_num_new_matched_tokens(3, prompt)}
    e.bind_pages(3, 96)
    e.update_state_after_alloc(3, 6, 4)
    m = e.build_connector_meta([(3, prompt)])
    out["cleared"] = e.store_clear(keys[1])
    transfer(e, m, 3, prompt)
    out["loaded"] = e.loaded_tokens(m, 3)
    out["pages_ok"] = pages_equal_synth(e, 3, prompt, 96, C)
    e.finish_query(3)
    e.release_query(3)
    e.close()
    return out


def sc_tier_full(factory, C):
    """test_connector.cpp:429-461: one slot, pinned stores -> one ok, one tier_full."""
    e = factory(**CONN, ram_slots=1, num_pages=64, pin_stores=True)
    prompt = make_prompt(64, 41)
    out = {"match": e.get_num_new_matched_tokens(4, prompt)}
    e.bind_pages(4, 64)
    out["upd"] = e.update_state_after_alloc(4, 4, 0)
    m = e.build_connector_meta([(4, prompt)])
    out["n_store"] = len(e.plan(m, 0, "store")[0])
    transfer(e, m, 4, prompt)
    codes = sorted(c for _, c in e.store_results(m, 4))
    out["codes"] = codes  # [0 (ok), 2 (tier_full)]
    e.finish_query(4)
    e.release_query(4)
    e.close()
    return out


def sc_degrade_blocking(factory, C):
    """test_connector.cpp:463-490: over-budget batch degrades to blocking."""
    e = factory(**CONN, ram_slots=16, num_pages=64, staging_budget=100)
    prompt = make_prompt(64, 43)
    e.seed_store(prompt, 64)
    out = {"match": e.get_num_new_matched_tokens(8, prompt)}
    e.bind_pages(8, 64)
    out["upd"] = e.update_state_after_alloc(8, 4, 4)
    m = e.build_connector_meta([(8, prompt)])
    out["mode_before"] = e.meta_layerwise(m)
    out["start"] = e.start_load_kv(m)
    out["mode_after"] = e.meta_layerwise(m)
    loaded = e.loaded_tokens(m, 8)
    out["loaded"] = loaded
    e.compute_range(8, prompt, loaded, len(prompt))
    out["store"] = e.start_store_kv(m)
    out["pages_ok"] = pages_equal_synth(e, 8, prompt, 64, C)
    e.finish_query(8)
    e.release_query(8)
    e.close()
    return out


def sc_multi_query_batch(factory, C):
    """Several queries in one scheduling iteration (SchedulerOutput with
    multiple queries): mixed warm / partial / cold, one metadata."""
    e = factory(**CONN, ram_slots=32, num_pages=256)
    prompts = {10: make_prompt(96, 101), 11: make_prompt(70, 102), 12: make_prompt(50, 103)}
    e.seed_store(prompts[10], 96)
    e.seed_store(prompts[11], 32)
    out = {}
    for q, p in prompts.items():
        out[f"match{q}"] = e.get_num_new_matched_tokens(q, p)
        e.bind_pages(q, len(p))
        blocks = (len(p) + 15) // 16
        e.update_state_after_alloc(q, blocks, (out[f"match{q}"] + 15) // 16)
    m = e.build_connector_meta(list(prompts.items()))
    for i, q in enumerate(prompts):
        out[f"plan{q}"] = plan_view(e, m, i)
    # Engine order for a batch: every query's layer computed, then stores.
    assert e.start_load_kv(m) == 0
    layerwise = e.meta_layerwise(m)
    for layer in range(e.num_layers):
        if layerwise:
            assert e.wait_load_kv(m, layer) == 0
        for q, p in prompts.items():
            lo = e.loaded_tokens(m, q)
            if hasattr(e, "stream_handle"):
                e.compute_range(q, p, lo, len(p), layers=(layer, layer + 1))
            else:
                e.compute_range(q, p, lo, len(p))
        if layer > 0:
            assert e.wait_store_kv(m, layer - 1) == 0
        assert e.start_store_kv(m) == 0
    assert e.wait_store_kv(m, e.num_layers - 1) == 0
    for q, p in prompts.items():
        out[f"loaded{q}"] = e.loaded_tokens(m, q)
        out[f"ok{q}"] = pages_equal_synth(e, q, p, len(p), C)
        out[f"res{q}"] = [(d.hex(), c) for d, c in e.store_results(m, q)]
        e.finish_query(q)
        e.release_query(q)
    out["entries"] = e.store_entries()
    e.close()
    return out


ALL = [sc_match_cap, sc_load_plan_clip, sc_inconsistent_alloc, sc_partial_match, sc_layerwise_vs_blocking,
       sc_vanishing_chunk, sc_tier_full, sc_degrade_blocking, sc_multi_query_batch]


def _random_trace(factory, C, seed: int, slots: int, decode: bool = False, probe: bool = False,
                  chunk_size: int = 32, scale: int = 1, num_pages: int = 1024, bpt: int = 64, layers: int = 4,
                  width: tuple = (1, 4), **cfg):
    """Randomised serving trace: shared document prefixes cut at arbitrary
    (non chunk- or page-aligned) points plus fresh tails, 1-3 queries per
    scheduling iteration, a RAM tier of `slots` chunks (small -> LRU evictions
    between iterations). Records every observable per query."""
    rng = np.random.default_rng(seed)
    geom = dict(CONN, chunk_size=chunk_size, bpt=bpt, num_layers=layers)
    e = factory(**geom, ram_slots=slots, num_pages=num_pages, **cfg)
    docs = [make_prompt(int(rng.integers(40, 200)) * scale, 1000 + 10 * seed + i) for i in range(4)]
    out = []
    qid = 100
    seen: set[str] = set()
    for _ in range(8):
        batch = []
        for _ in range(int(rng.integers(*width))):
            d = docs[int(rng.integers(0, len(docs)))]
            cut = int(rng.integers(1, len(d) + 1))
            tail = make_prompt(int(rng.integers(0, 40)), int(rng.integers(0, 1 << 30)))
            batch.append((qid, np.concatenate([d[:cut], tail]).astype(np.uint32)))
            qid += 1
        n_dec = {q: int(rng.integers(0, 70)) if decode and rng.random() < 0.6 else 0 for q, _ in batch}
        rec = {"matched": [e.get_num_new_matched_tokens(q, p) for q, p in batch]}
        for (q, p), mt in zip(batch, rec["matched"]):
            n_all = len(p) + n_dec[q]
            e.bind_pages(q, n_all)
            assert e.update_state_after_alloc(q, (n_all + 15) // 16, (mt + 15) // 16) == 0
        m = e.build_connector_meta(batch)
        rec["plans"] = [plan_view(e, m, i) for i in range(len(batch))]
        assert e.start_load_kv(m) == 0
        layerwise = e.meta_layerwise(m)
        for layer in range(e.num_layers):
            if layerwise:
                assert e.wait_load_kv(m, layer) == 0
            for q, p in batch:
                lo = e.loaded_tokens(m, q)
                if hasattr(e, "stream_handle"):
                    e.compute_range(q, p, lo, len(p), layers=(layer, layer + 1))
                else:
                    e.compute_range(q, p, lo, len(p))
            if layerwise:
                if layer > 0:
                    assert e.wait_store_kv(m, layer - 1) == 0
                assert e.start_store_kv(m) == 0
        if layerwise:
            assert e.wait_store_kv(m, e.num_layers - 1) == 0
        else:  # blocking: one store of every layer after the compute (sim_engine.cpp:150-160)
            assert e.start_store_kv(m) == 0
        rec["loaded"] = [e.loaded_tokens(m, q) for q, _ in batch]
        rec["pages_ok"] = [pages_equal_synth(e, q, p, len(p), C) for q, p in batch]
        rec["results"] = [[(d.hex(), c) for d, c in e.store_results(m, q)] for q, _ in batch]
        seen = {d for r in rec["results"] for d, _ in r} | seen
        if probe:  # diagnostics: which chunks the tier holds after the batch
            rec["present_after_batch"] = sorted(d[:8] for d in seen if e.contains(bytes.fromhex(d)))
            # decode storing (connector.cpp:434-497): generated tokens' KV
            # computed one at a time, full chunks flushed as they complete,
            # the tail at finish_query
            rec["decode"] = []
            for q, p in batch:
                if not n_dec[q]:
                    rec["decode"].append(None)
                    continue
                gen = make_prompt(n_dec[q], int(rng.integers(0, 1 << 30)))
                full = np.concatenate([p, gen]).astype(np.uint32)
                rcs = [e.begin_decode(q)]
                for i, tok in enumerate(gen):
                    e.compute_range(q, full, len(p) + i, len(p) + i + 1)
                    rcs.append(e.append_decode(q, int(tok)))
                keys, rc = e.finish_query_keys(q)
                rec["decode"].append({"rcs": rcs, "keys": [k.hex() for k in keys], "rc": rc})
                if probe:
                    seen |= {k.hex() for k in keys}
                    rec["decode"][-1]["present"] = sorted(d[:8] for d in seen if e.contains(bytes.fromhex(d)))
        for q, _ in batch:
            e.finish_query(q)
            e.release_query(q)
        rec["entries"] = e.store_entries()
        out.append(rec)
    e.close()
    return out


def sc_random_trace_roomy(factory, C):
    """Random trace, tier large enough to keep everything."""
    return [_random_trace(factory, C, seed, 256) for seed in (1, 2, 3)]


def sc_random_trace_evicting(factory, C):
    """Random trace, 6-chunk tier: LRU evictions decide later hits."""
    return [_random_trace(factory, C, seed, 6) for seed in (4, 5, 6)]


def sc_random_trace_pinned(factory, C):
    """Random trace, pinned stores into an 8-chunk tier: fills, then tier_full."""
    return [_random_trace(factory, C, seed, 8, pin_stores=True) for seed in (7, 8)]


def sc_random_trace_blocking(factory, C):
    """Random trace in blocking (non-layerwise) mode with evictions."""
    return [_random_trace(factory, C, seed, 5, layerwise=False) for seed in (9, 10)]


def sc_random_trace_decode(factory, C):
    """Random trace with decode storing after each prefill, roomy and evicting tiers."""
    return [_random_trace(factory, C, 11, 256, decode=True), _random_trace(factory, C, 12, 7, decode=True)]


def sc_random_trace_big_chunks(factory, C):
    """Random trace with 512-token chunks (the thread-per-chain K3 variant and
    32-page chunk spans) and 1K-3K-token documents, evicting tier."""
    return [_random_trace(factory, C, 13, 10, chunk_size=512, scale=16, num_pages=12000)]


def sc_random_trace_odd_rows(factory, C):
    """Random trace with 12- and 40-byte rows (4- and 8-byte vector paths of
    K1/K2, byte tails in synth) and 3 / 5 layers, evicting tier."""
    return [_random_trace(factory, C, 14, 6, bpt=12, layers=3), _random_trace(factory, C, 15, 6, bpt=40, layers=5)]


def sc_random_trace_wide(factory, C):
    """Random trace with 5-12 queries per scheduling iteration (many plans,
    shared chunks across queries of one batch), roomy and evicting tiers."""
    return [_random_trace(factory, C, 16, 256, width=(5, 13), num_pages=4096),
            _random_trace(factory, C, 17, 12, width=(5, 13), num_pages=4096)]


ALL += [sc_random_trace_roomy, sc_random_trace_evicting, sc_random_trace_pinned, sc_random_trace_blocking,
        sc_random_trace_decode, sc_random_trace_big_chunks, sc_random_trace_odd_rows, sc_random_trace_wide]


def sc_degenerate_prompts(factory, C):
    """Edge lengths through the whole connector sequence: 1 token, exactly one
    chunk, one chunk + 1, a chunk minus 1, a page exactly, and an empty
    lookup (cap min(lpm, len - 1), connector.cpp:75-76)."""
    e = factory(**CONN, ram_slots=32, num_pages=256)
    out = {"empty": e.get_num_new_matched_tokens(1, np.zeros(0, np.uint32))}
    qid = 10
    for n in (1, 32, 33, 31, 16):
        p = make_prompt(n, 500 + n)
        for rnd in range(2):  # cold store, then warm retrieve of the same prompt
            mt = e.get_num_new_matched_tokens(qid, p)
            e.bind_pages(qid, n)
            upd = e.update_state_after_alloc(qid, (n + 15) // 16, (mt + 15) // 16)
            m = e.build_connector_meta([(qid, p)])
            transfer(e, m, qid, p)
            out[f"n{n}_r{rnd}"] = {"matched": mt, "upd": upd, "plan": plan_view(e, m, 0),
                                   "loaded": e.loaded_tokens(m, qid),
                                   "ok": pages_equal_synth(e, qid, p, n, C),
                                   "res": [(d.hex(), c) for d, c in e.store_results(m, qid)]}
            e.finish_query(qid)
            e.release_query(qid)
            qid += 1
    out["entries"] = e.store_entries()
    e.close()
    return out


ALL += [sc_degenerate_prompts]


def sc_api_errors(factory, C):
    """Error behaviour of the connector calls (connector.cpp:239-392,
    434-497): layer out of range, a store wait before its start, surplus
    store starts, decode on an unplanned query, finish of an unknown query."""
    e = factory(**CONN, ram_slots=16, num_pages=64)
    prompt = make_prompt(70, 31)
    e.seed_store(prompt, 32)
    out = {"match": e.get_num_new_matched_tokens(7, prompt)}
    e.bind_pages(7, 70)
    out["upd"] = e.update_state_after_alloc(7, 5, 2)
    m = e.build_connector_meta([(7, prompt)])
    out["start_load"] = e.start_load_kv(m)
    out["wait_load_out_of_range"] = e.wait_load_kv(m, e.num_layers)
    out["wait_store_out_of_range"] = e.wait_store_kv(m, e.num_layers)
    out["wait_store_not_started"] = e.wait_store_kv(m, 0)
    loaded = e.loaded_tokens(m, 7)
    starts = []
    for layer in range(e.num_layers):
        assert e.wait_load_kv(m, layer) == 0
        if hasattr(e, "stream_handle"):
            e.compute_range(7, prompt, loaded, 70, layers=(layer, layer + 1))
        else:
            e.compute_range(7, prompt, loaded, 70)
        starts.append(e.start_store_kv(m))
    starts.append(e.start_store_kv(m))  # one more than there are layers
    out["starts"] = starts
    out["final_wait"] = e.wait_store_kv(m, e.num_layers - 1)
    out["final_wait_again"] = e.wait_store_kv(m, e.num_layers - 1)
    out["results"] = [(d.hex(), c) for d, c in e.store_results(m, 7)]
    out["pages_ok"] = pages_equal_synth(e, 7, prompt, 70, C)
    out["decode_unplanned"] = e.begin_decode(12345)
    out["finish_unknown"] = e.finish_query(999)
    out["finish"] = e.finish_query(7)
    e.release_query(7)
    e.close()
    return out


ALL += [sc_api_errors]


def _store_op_soup(factory, seed: int, n_ops: int, ram_slots: int, n_keys: int):
    """Sequential random RAM-tier operations straight on the store
    (test_store.cpp: put/get round trips, duplicate puts, LRU eviction that
    spares pinned entries and reports tier_full when stuck, clear refusing
    pinned copies, pin of an absent key, per-layer reads). Every result is
    logged; payloads by digest."""
    import hashlib
    e = factory(num_layers=3, bpt=24, page_tokens=16, tag="soup", chunk_size=32, ram_slots=ram_slots,
                num_pages=16)
    rng = np.random.default_rng(seed)
    keys = [rng.integers(0, 256, 32, dtype=np.uint8).tobytes() for _ in range(n_keys)]
    h = (lambda b: None if b is None else hashlib.sha256(b.tobytes()).hexdigest()[:16])
    log = []
    for _ in range(n_ops):
        k = keys[int(rng.integers(n_keys))]
        op = int(rng.integers(8))
        if op <= 2:
            tc = int(rng.choice([32, 32, 32, 17, 1]))
            pay = rng.integers(0, 256, 3 * tc * 24, dtype=np.uint8)
            log.append(("put", tc, e.store_put(k, tc, pay, bool(rng.random() < 0.15))))
        elif op == 3:
            log.append(("get", h(e.store_get(k))))
        elif op == 4:
            layer = int(rng.integers(4))  # 3 = out of range
            code, b = e.store_get_layer(k, layer)
            log.append(("get_layer", layer, code, h(b)))
        elif op == 5:
            log.append(("pin", e.store_pin(k, bool(rng.random() < 0.6))))
        elif op == 6:
            log.append(("clear", *e.store_clear_n(k)))
        else:
            log.append(("contains", e.contains(k), *e.store_stats()))
    log.append(("final", *e.store_stats()))
    e.close()
    return log


def sc_store_op_soup(factory, C):
    """RAM-tier op soup: 6 and 3 slots over 12 and 8 keys (evictions, pinned
    slots, tier_full), one and two slots, and a roomy tier."""
    return [_store_op_soup(factory, 1, 400, 6, 12), _store_op_soup(factory, 2, 400, 3, 8),
            _store_op_soup(factory, 3, 300, 64, 12), _store_op_soup(factory, 4, 300, 1, 5),
            _store_op_soup(factory, 5, 300, 2, 6)]


ALL += [sc_store_op_soup]


def _protocol_fuzz(factory, C, seed: int):
    """Serving iterations with protocol slips mixed in, every return code
    logged (connector.cpp:71-164, 239-392): allocation updates with wrong
    block counts before the right one, a second lookup of a query with a
    different prompt, queries planned without a lookup or without an
    allocation update, out-of-range and early waits, surplus store starts,
    finish of unknown queries."""
    rng = np.random.default_rng(seed)
    e = factory(**CONN, ram_slots=12, num_pages=1024)
    docs = [make_prompt(int(rng.integers(40, 160)), 3000 + 10 * seed + i) for i in range(3)]
    log = []
    qid = 500
    for _ in range(10):
        batch = []
        for _ in range(int(rng.integers(1, 4))):
            d = docs[int(rng.integers(0, len(docs)))]
            cut = int(rng.integers(1, len(d) + 1))
            p = np.concatenate([d[:cut], make_prompt(int(rng.integers(0, 30)), int(rng.integers(1 << 30)))])
            batch.append((qid, p.astype(np.uint32)))
            qid += 1
        rec = {}
        slip = {q: int(rng.integers(0, 6)) for q, _ in batch}
        matched = {}
        for q, p in batch:
            if slip[q] == 1:  # looked up once with another prompt first
                rec[f"pre{q}"] = e.get_num_new_matched_tokens(q, make_prompt(len(p) + 7, q))
            matched[q] = e.get_num_new_matched_tokens(q, p) if slip[q] != 2 else None
        for q, p in batch:
            e.bind_pages(q, len(p))
            ext = (matched[q] or 0) + 15
            ext //= 16
            blocks = (len(p) + 15) // 16
            if slip[q] == 3:  # wrong counts first
                rec[f"bad_ext{q}"] = e.update_state_after_alloc(q, blocks, ext + 1)
                if blocks:
                    rec[f"bad_blocks{q}"] = e.update_state_after_alloc(q, max(0, ext - 1), ext)
            if slip[q] != 4:
                rec[f"upd{q}"] = e.update_state_after_alloc(q, blocks, ext)
        m = e.build_connector_meta(batch)
        rec["plans"] = [plan_view(e, m, i) for i in range(len(batch))]
        rec["start_load"] = e.start_load_kv(m)
        layerwise = e.meta_layerwise(m)
        rec["early_store_wait"] = e.wait_store_kv(m, 0)
        rec["wait_load_oob"] = e.wait_load_kv(m, e.num_layers + int(rng.integers(0, 3)))
        for layer in range(e.num_layers):
            if layerwise:
                rec[f"wl{layer}"] = e.wait_load_kv(m, layer)
            for q, p in batch:
                lo = e.loaded_tokens(m, q)
                if hasattr(e, "stream_handle"):
                    e.compute_range(q, p, lo, len(p), layers=(layer, layer + 1))
                else:
                    e.compute_range(q, p, lo, len(p))
            if layerwise:
                if layer > 0:
                    rec[f"ws{layer - 1}"] = e.wait_store_kv(m, layer - 1)
                rec[f"ss{layer}"] = e.start_store_kv(m)
        if layerwise:
            if rng.random() < 0.3:
                rec["surplus_start"] = e.start_store_kv(m)
            rec["final"] = e.wait_store_kv(m, e.num_layers - 1)
        else:
            rec["blocking_store"] = e.start_store_kv(m)
        rec["loaded"] = [e.loaded_tokens(m, q) for q, _ in batch]
        rec["pages_ok"] = [pages_equal_synth(e, q, p, len(p), C) for q, p in batch]
        rec["results"] = [[(d.hex(), c) for d, c in e.store_results(m, q)] for q, _ in batch]
        rec["finish_unknown"] = e.finish_query(qid + 1000)
        rec["finish"] = [e.finish_query(q) for q, _ in batch]
        rec["finish_again"] = [e.finish_query(q) for q, _ in batch]
        for q, _ in batch:
            e.release_query(q)
        rec["entries"] = e.store_entries()
        log.append(rec)
    e.close()
    return log


def sc_protocol_fuzz(factory, C):
    return [_protocol_fuzz(factory, C, seed) for seed in (1, 2, 3, 4)]


ALL += [sc_protocol_fuzz]


def _prefill(e, C, q, p, extra):
    """One query through a full layerwise (or blocking) iteration, pages for
    len(p) + extra tokens."""
    mt = e.get_num_new_matched_tokens(q, p)
    n_all = len(p) + extra
    e.bind_pages(q, n_all)
    rc = e.update_state_after_alloc(q, (n_all + 15) // 16, (mt + 15) // 16)
    m = e.build_connector_meta([(q, p)])
    transfer(e, m, q, p)
    out = {"matched": mt, "upd": rc, "loaded": e.loaded_tokens(m, q),
           "res": [(d.hex(), c) for d, c in e.store_results(m, q)]}
    e.drop_meta(m)
    return out


def _decode_fuzz(factory, C, seed: int):
    """Decode storing (connector.cpp:434-497) with several queries decoding
    interleaved and protocol slips: begin twice, append before begin or
    after finish, finish twice. Logs every code, the flushed keys and the
    stored bytes of every flushed chunk."""
    import hashlib
    rng = np.random.default_rng(seed)
    e = factory(**CONN, ram_slots=32, num_pages=2048)
    log = []
    qs = {}
    for i in range(4):
        q = 900 + i
        p = make_prompt(int(rng.integers(1, 100)), 4000 + 10 * seed + i)
        log.append(("prefill", q, _prefill(e, C, q, p, 90)))
        qs[q] = {"p": p, "gen": [], "state": "prefilled"}
    for _ in range(260):
        q = 900 + int(rng.integers(0, 4))
        s = qs[q]
        r = rng.random()
        if s["state"] == "prefilled" and r > 0.3:
            r = 0.0  # mostly begin a prefilled query; sometimes slip an append first
        if r < 0.06:
            log.append(("begin", q, e.begin_decode(q)))
            if s["state"] == "prefilled":
                s["state"] = "decoding"
        elif r < 0.09:
            keys, rc = e.finish_query_keys(q)
            log.append(("finish", q, rc, [k.hex() for k in keys]))
            s["state"] = "finished"
        else:
            tok = int(rng.integers(0, 32000))
            if s["state"] == "decoding" and len(s["gen"]) < 90:
                full = np.concatenate([s["p"], np.array(s["gen"] + [tok], np.uint32)]).astype(np.uint32)
                pos = len(full) - 1
                e.compute_range(q, full, pos, pos + 1)
                rc = e.append_decode(q, tok)
                if rc == 0:
                    s["gen"].append(tok)
                log.append(("append", q, rc))
            elif s["state"] != "decoding":
                log.append(("append_slip", q, e.append_decode(q, tok)))
    for q, s in qs.items():
        keys, rc = e.finish_query_keys(q)
        log.append(("final_finish", q, rc, [k.hex() for k in keys]))
    # every chunk the decode flushed: its bytes in the tier
    h = (lambda b: None if b is None else hashlib.sha256(b.tobytes()).hexdigest()[:16])
    flushed = sorted({k for x in log if x[0] in ("finish", "final_finish") for k in x[-1]})
    log.append(("stored", [(k[:16], h(e.store_get(bytes.fromhex(k)))) for k in flushed]))
    for q in qs:
        e.release_query(q)
    e.close()
    return log


def sc_decode_fuzz(factory, C):
    return [_decode_fuzz(factory, C, seed) for seed in (1, 2, 3)]


ALL += [sc_decode_fuzz]


def _pipelined(factory, C, seed: int, n_req: int = 6, batch: int = 1):
    """Serving schedule with two scheduling iterations in flight (bench.py's
    run_pipelined): the B200 engine looks up and begins iteration k+1 — bind,
    plan, start_load_kv and every layer's wait_load / compute / start_store —
    before iteration k's final wait_store_kv; the reference runs the same
    iterations one after another (its sequential order, connector.cpp:239-392).
    Every iteration retrieves a shared stored document prefix and stores fresh
    suffixes of 3 chunks per query (ragged tails); the tier holds the prefix
    plus two iterations' suffixes, so each iteration's stores evict the
    suffixes of the iteration two back (LRU), while its predecessor's are still
    being written. Records every hit length, plan, loaded count, store status,
    page image and the payload of every chunk left in the tier."""
    rng = np.random.default_rng(seed)
    cs = CONN["chunk_size"]
    doc = make_prompt(3 * cs, 7000 + seed)  # 3 chunks, stored up front
    S = 3 * batch
    e = factory(**CONN, ram_slots=3 + 2 * S, num_pages=4096)
    e.seed_store(doc, len(doc))
    pipelined = hasattr(e, "stream_handle")
    iters = []
    for k in range(n_req):
        qs = []
        for b in range(batch):
            tail = make_prompt(2 * cs + int(rng.integers(1, cs + 1)), int(rng.integers(0, 1 << 30)))
            qs.append((1000 + batch * k + b, np.concatenate([doc, tail]).astype(np.uint32)))
        iters.append(qs)
    out = {"iters": []}

    def lookup(qs):
        return [e.get_num_new_matched_tokens(q, p) for q, p in qs]

    def begin(qs, matched):
        for (q, p), mt in zip(qs, matched):
            assert e.bind_pages(q, len(p)) == 0
            assert e.update_state_after_alloc(q, (len(p) + 15) // 16, (mt + 15) // 16) == 0
        m = e.build_connector_meta(qs)
        assert e.start_load_kv(m) == 0
        for layer in range(e.num_layers):
            assert e.wait_load_kv(m, layer) == 0
            for q, p in qs:
                lo = e.loaded_tokens(m, q)
                if pipelined:
                    e.compute_range(q, p, lo, len(p), layers=(layer, layer + 1))
                else:
                    e.compute_range(q, p, lo, len(p))
            if layer:
                assert e.wait_store_kv(m, layer - 1) == 0
            assert e.start_store_kv(m) == 0
        return m

    def end(qs, matched, m):
        assert e.wait_store_kv(m, e.num_layers - 1) == 0
        rec = {"matched": matched, "plans": [plan_view(e, m, i) for i in range(len(qs))],
               "loaded": [e.loaded_tokens(m, q) for q, _ in qs],
               "pages_ok": [pages_equal_synth(e, q, p, len(p), C) for q, p in qs],
               "image": [page_image(e, q, len(p)) for q, p in qs],
               "results": [[(d.hex(), c) for d, c in e.store_results(m, q)] for q, _ in qs]}
        e.drop_meta(m)
        for q, _ in qs:
            e.finish_query(q)
            if pipelined:
                e.release_query(q, sync=False)  # the next iteration stays in flight
            else:
                e.release_query(q)
        out["iters"].append(rec)

    if pipelined:
        mt = lookup(iters[0])
        cur = (iters[0], mt, begin(iters[0], mt))
        for k in range(n_req):
            nxt = None
            if k + 1 < n_req:
                mt = lookup(iters[k + 1])
                nxt = (iters[k + 1], mt, begin(iters[k + 1], mt))
            end(*cur)
            cur = nxt
    else:
        for qs in iters:
            mt = lookup(qs)
            end(qs, mt, begin(qs, mt))
    # every chunk any iteration stored: still in the tier? its bytes
    seed_m = C.model_seed(e.tag)
    tier = []
    for qs in iters:
        for q, p in qs:
            keys = C.chunk_keys(p, cs, e.tag)
            for i in range(3, len(keys)):
                got = e.store_get(keys[i])
                if got is None:
                    tier.append((keys[i].hex()[:16], None))
                else:
                    cnt = min(cs, len(p) - cs * i)
                    want = C.synth_chunk(seed_m, p, cs * i, cnt, e.num_layers, e.bpt)
                    tier.append((keys[i].hex()[:16], bool(np.array_equal(got, want))))
    out["tier"] = tier
    out["entries"] = e.store_entries()
    e.close()
    return out


def sc_pipelined_two_in_flight(factory, C):
    """Two iterations in flight (B200) vs sequential (reference): one query per
    iteration, and three queries per iteration (one plan per query, 9 suffix
    chunks per iteration)."""
    return [_pipelined(factory, C, 1), _pipelined(factory, C, 2, n_req=5, batch=3)]


ALL += [sc_pipelined_two_in_flight]
