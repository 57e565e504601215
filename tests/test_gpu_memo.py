"""The device prefix-digest memo never changes a
key: every digest the connector plans with equals the CPU oracle's chain,
whether it came from SHA or from a verified memo hit — for repeated prompts,
shared prefixes, equal chunk contents under different parents, partial tails,
and a memo small enough to fill up and reset."""
import numpy as np
import pytest

import scenarios as S

pytestmark = pytest.mark.gpu

TAG = "memo-test"


def _keys_via_connector(e, qid, prompt):
    """Digests the connector derived for `prompt` (nothing stored -> the store
    plan lists every chunk with its key)."""
    e.get_num_new_matched_tokens(qid, prompt)
    e.bind_pages(qid, len(prompt))
    e.update_state_after_alloc(qid, (len(prompt) + 15) // 16, 0)
    m = e.build_connector_meta([(qid, prompt)])
    sp, _ = e.plan(m, 0, "store")
    e.drop_meta(m)
    e.finish_query(qid)
    e.release_query(qid)
    return [d for _, _, _, _, d in sp]


@pytest.mark.parametrize("entries", [65536, 24])
def test_memo_keys_equal_oracle(tkv, C, entries):
    from paper_2510_09665_b200.api import Engine
    e = Engine(num_layers=2, bpt=64, page_tokens=16, tag=TAG, chunk_size=256, ram_slots=2, num_pages=4096,
               memo_entries=entries)
    rng = np.random.default_rng(entries)
    doc = rng.integers(0, 128256, size=256 * 12, dtype=np.uint32)
    prompts = [doc, doc.copy(),                                   # repeat: all hits
               np.concatenate([doc[:256 * 5], rng.integers(0, 128256, 300, dtype=np.uint32)]),  # shared prefix
               np.concatenate([doc[256:512], doc[:256], doc[512:900]]),  # same chunk bytes, other parents
               doc[:256 * 3 + 17],                                # partial tail
               doc]
    qid = 1
    for p in prompts:
        assert _keys_via_connector(e, qid, p) == C.chunk_keys(p, 256, TAG)
        qid += 1
    st = e.memo_stats()
    if entries == 65536:
        assert st["hits"] >= 12 + 12 + 5 + 3 and st["resets"] == 0
    else:
        assert st["resets"] >= 1
    e.close()


def test_memo_false_hit_is_caught_and_rehashed(tkv, C):
    """Corrupt every memo slot's digest: the optimistic chain then follows a
    wrong digest, the parallel verification must flag it and the chain must be
    re-hashed, giving the oracle keys."""
    from paper_2510_09665_b200.api import Engine
    e = Engine(num_layers=2, bpt=64, page_tokens=16, tag=TAG, chunk_size=256, ram_slots=2, num_pages=4096)
    rng = np.random.default_rng(42)
    doc = rng.integers(0, 128256, size=256 * 9 + 40, dtype=np.uint32)
    assert _keys_via_connector(e, 1, doc) == C.chunk_keys(doc, 256, TAG)
    e.debug_poison_memo()
    before = e.memo_stats()["rehashes"]
    assert _keys_via_connector(e, 2, doc) == C.chunk_keys(doc, 256, TAG)
    assert e.memo_stats()["rehashes"] == before + 1
    e.close()


def test_memo_does_not_change_connector_outcomes(tkv, C):
    """The connector scenarios give the reference outcome with the memo on
    (default) and off."""
    import json

    from paper_2510_09665_b200.api import Engine
    for name in ("sc_partial_match", "sc_multi_query_batch"):
        on = json.loads(json.dumps(getattr(S, name)(Engine, C)))
        off = json.loads(json.dumps(getattr(S, name)(
            lambda **kw: Engine(**kw, memo_entries=0), C)))
        assert on == off


def test_memo_batched_mixed_hits(tkv, C):
    """One lookup launch over many chains: full hits, a shared prefix that
    diverges mid-chain, a cold chain, a repeat inside the batch and a partial
    tail. The parallel probes resume each chain at its own first miss."""
    from paper_2510_09665_b200.api import Engine
    e = Engine(num_layers=2, bpt=64, page_tokens=16, tag=TAG, chunk_size=256, ram_slots=2, num_pages=8192)
    rng = np.random.default_rng(7)
    doc = rng.integers(0, 128256, size=256 * 20 + 33, dtype=np.uint32)
    assert _keys_via_connector(e, 1, doc) == C.chunk_keys(doc, 256, TAG)  # warm the memo
    cold = rng.integers(0, 128256, size=256 * 7, dtype=np.uint32)
    diverge = doc.copy()
    diverge[256 * 9 + 100] ^= 1
    prompts = [doc, diverge, cold, doc[:256 * 4 + 5], cold, doc[:256 * 20]]
    ids = list(range(10, 10 + len(prompts)))
    e.lookup_batch(ids, prompts)
    for q, p in zip(ids, prompts):
        e.bind_pages(q, len(p))
        e.update_state_after_alloc(q, (len(p) + 15) // 16, 0)
    m = e.build_connector_meta(list(zip(ids, prompts)))
    for i, p in enumerate(prompts):
        sp, _ = e.plan(m, i, "store")
        assert [d for _, _, _, _, d in sp] == C.chunk_keys(p, 256, TAG), i
    e.drop_meta(m)
    st = e.memo_stats()
    # doc: 21 hits; diverge: 9; doc[:4 full + 5]: 4; doc[:20 full]: 20
    assert st["hits"] >= 21 + 9 + 4 + 20
    assert st["rehashes"] == 0
    e.close()


def test_memo_resumed_chain_parent(tkv, C):
    """KeyChain::next with a parent (tokens.hpp:41-63) through the memo-enabled
    free-function hasher: equal chunk tokens under different parents never
    share a link, and a repeated (parent, chunk) is served from the memo."""
    from paper_2510_09665_b200.api import chunk_keys, keychain_next
    rng = np.random.default_rng(9)
    chunk = rng.integers(0, 128256, size=256, dtype=np.uint32)
    parents = [bytes(32), bytes(range(32)), bytes(31) + b"\x01"]
    for _ in range(2):
        for p in parents:
            assert keychain_next(TAG, 256, p, chunk) == C.keychain_next(TAG, p, chunk)
    doc = rng.integers(0, 128256, size=256 * 6 + 7, dtype=np.uint32)
    for _ in range(2):
        assert chunk_keys(doc, 256, TAG) == C.chunk_keys(doc, 256, TAG)


def test_memo_batch_with_empty_and_single_token_prompts(tkv, C):
    """Empty and one-token prompts in the same lookup launch as long ones
    (zero-row chains next to multi-row chains in the probe and hash kernels)."""
    from paper_2510_09665_b200.api import Engine
    e = Engine(num_layers=2, bpt=64, page_tokens=16, tag=TAG, chunk_size=256, ram_slots=2, num_pages=4096)
    rng = np.random.default_rng(3)
    doc = rng.integers(0, 128256, size=256 * 3 + 9, dtype=np.uint32)
    one = doc[:1].copy()
    empty = np.zeros(0, np.uint32)
    for rnd in range(2):  # cold memo, then warm
        got = e.lookup_batch([10 * rnd + 1, 10 * rnd + 2, 10 * rnd + 3, 10 * rnd + 4], [empty, doc, one, empty])
        assert got == [0, 0, 0, 0]  # nothing stored: no hits
        keys = []
        for q, p in zip([10 * rnd + 2, 10 * rnd + 3], [doc, one]):
            e.bind_pages(q, len(p))
            e.update_state_after_alloc(q, (len(p) + 15) // 16, 0)
            m = e.build_connector_meta([(q, p)])
            sp, _ = e.plan(m, 0, "store")
            keys.append([d for _, _, _, _, d in sp])
            e.drop_meta(m)
        assert keys == [C.chunk_keys(doc, 256, TAG), C.chunk_keys(one, 256, TAG)]
        for q in range(10 * rnd + 1, 10 * rnd + 5):
            e.finish_query(q)
            e.release_query(q)
    assert e.memo_stats()["rehashes"] == 0
    e.close()


def test_prefix_lookups_do_not_fill_the_memo(tkv, C):
    """A lookup inserts at most one link per chain (the first absent chunk),
    so many lookups of one stored document under new questions keep the memo
    warm: no reset, and every lookup still matches the whole document."""
    from paper_2510_09665_b200.api import Engine
    e = Engine(num_layers=1, bpt=64, page_tokens=16, tag=TAG, chunk_size=256, ram_slots=48, num_pages=64,
               memo_entries=256)
    rng = np.random.default_rng(9)
    doc = rng.integers(0, 128256, size=256 * 40, dtype=np.uint32)
    e.seed_store(doc, len(doc))
    for q in range(100):  # 100 lookups x 41 chunks would overflow a 256-entry bound 16 times
        p = np.concatenate([doc, rng.integers(0, 128256, 60, dtype=np.uint32)])
        assert e.get_num_new_matched_tokens(q + 1, p) == len(doc)
        e.finish_query(q + 1)
    st = e.memo_stats()
    assert st["resets"] == 0 and st["hits"] >= 99 * 40
    e.close()


@pytest.mark.parametrize("n_queries", [127, 129, 300])
def test_memo_many_chains_one_launch(tkv, C, n_queries):
    """Lookups and planning over more chains than the fingerprint pass stages
    per block (128): descriptors come through the separate copy, keys still
    equal the oracle's; below the limit they are staged in the same launch."""
    from paper_2510_09665_b200.api import Engine
    e = Engine(num_layers=1, bpt=16, page_tokens=16, tag=TAG, chunk_size=32, ram_slots=4, num_pages=20000)
    rng = np.random.default_rng(n_queries)
    doc = rng.integers(0, 128256, size=32 * 6, dtype=np.uint32)
    prompts = [np.concatenate([doc[:int(rng.integers(0, len(doc)))],
                               rng.integers(0, 128256, size=int(rng.integers(0, 70)), dtype=np.uint32)])
               for _ in range(n_queries)]
    ids = list(range(1, n_queries + 1))
    e.lookup_batch(ids, prompts)
    for q, p in zip(ids, prompts):
        e.bind_pages(q, max(1, len(p)))
        e.update_state_after_alloc(q, (len(p) + 15) // 16, 0)
    m = e.build_connector_meta(list(zip(ids, prompts)))
    for i, p in enumerate(prompts):
        sp, _ = e.plan(m, i, "store")
        assert [d for _, _, _, _, d in sp] == C.chunk_keys(p, 32, TAG), i
    e.drop_meta(m)
    e.close()


def test_presence_index_decides_lookups_on_device(tkv, C):
    """The stored prefix is decided in the lookup launches from the device
    presence index (TieredStore's present set mirrored in mapped memory):
    warm, partially stored, evicted, cleared and cold prompts give the
    reference's hit lengths with no host presence probe; a chunk stored
    without a memo link (seeded straight into the tier) and a memo whose
    hits fail verification fall back to the host index and still agree."""
    from paper_2510_09665_b200.api import Engine
    rng = np.random.default_rng(3)
    e = Engine(num_layers=2, bpt=64, page_tokens=16, tag=TAG, chunk_size=256, ram_slots=6, num_pages=4096)
    doc = rng.integers(0, 128256, size=256 * 5 + 40, dtype=np.uint32)
    keys = C.chunk_keys(doc, 256, TAG)

    def lookup(qid, p):
        m = e.get_num_new_matched_tokens(qid, p)
        e.finish_query(qid)
        return m

    def store(qid, p):  # a cold prefill through the connector (memo links + tier entries)
        e.get_num_new_matched_tokens(qid, p)
        e.bind_pages(qid, len(p))
        e.update_state_after_alloc(qid, (len(p) + 15) // 16, 0)
        m = e.build_connector_meta([(qid, p)])
        S.transfer(e, m, qid, p)
        e.drop_meta(m)
        e.finish_query(qid)
        e.release_query(qid)

    assert lookup(1, doc) == 0                       # cold: chunk 0 hashed, absent
    store(2, doc)                                     # all 6 chunks stored (tier full)
    base = e.lookups_host_decided()
    assert lookup(3, doc) == len(doc) - 1             # warm: every row a memo hit, all present
    assert lookup(4, doc[:256 * 3 + 7]) == 256 * 3    # shared prefix, new tail
    assert e.store_clear(keys[2]) == 1                # a present memo hit that left the tier
    assert lookup(5, doc) == 512
    assert e.lookups_host_decided() == base
    other = rng.integers(0, 128256, size=256 * 2, dtype=np.uint32)
    store(6, other)                                   # LRU evicts the oldest two of doc's chunks
    want = 0 if not e.contains(keys[0]) else (256 if not e.contains(keys[1]) else 512)
    assert lookup(7, doc) == want
    assert lookup(8, other) == 511
    assert e.lookups_host_decided() == base
    # stored chunks the memo never linked: the first-row kernel links chunk 0,
    # chunk 1 is hashed and present too, so the device cannot decide chunk 2
    # and the host continues the chain
    fresh = rng.integers(0, 128256, size=256 * 3, dtype=np.uint32)
    e.seed_store(fresh, 768)                          # tier entries without memo links
    assert lookup(9, fresh) == 767
    assert e.lookups_host_decided() == base + 1
    e.close()


def test_presence_many_changes_between_lookups(tkv, C):
    """Thousands of presence changes between two lookups (a tier filled by
    one large store, then an evicting one): the change feed grows its index,
    coalesces, and the next lookups — cold (first-row kernel, the changes
    applied in that launch) and warm (the fingerprint pass applies them) —
    still equal the host index."""
    from paper_2510_09665_b200.api import Engine
    rng = np.random.default_rng(11)
    e = Engine(num_layers=1, bpt=16, page_tokens=16, tag=TAG, chunk_size=256, ram_slots=1500, num_pages=8192)
    big = rng.integers(0, 128256, size=256 * 1400, dtype=np.uint32)
    e.seed_store(big, len(big))                     # 1400 adds
    cold = rng.integers(0, 128256, size=256 * 3, dtype=np.uint32)
    assert e.get_num_new_matched_tokens(1, cold) == 0
    e.finish_query(1)
    other = rng.integers(0, 128256, size=256 * 300, dtype=np.uint32)
    e.seed_store(other, len(other))                 # 300 adds, 200 evictions
    assert e.get_num_new_matched_tokens(2, rng.integers(0, 128256, size=600, dtype=np.uint32)) == 0
    e.finish_query(2)
    keys = C.chunk_keys(big, 256, TAG)
    want = 0
    while want < len(keys) and e.contains(keys[want]):
        want += 1
    assert e.get_num_new_matched_tokens(3, big) == min(len(big) - 1, 256 * want)
    e.finish_query(3)
    assert e.get_num_new_matched_tokens(4, other) == len(other) - 1
    e.finish_query(4)
    e.close()


def test_absence_witness_decides_without_sha(tkv, C):
    """The absence witness (kernels.hpp PresenceView): a row whose prefix key
    no present digest has is absent without its SHA-256 — the cold first row
    of a new document (first-row kernel) and the question row after a stored
    document (probe kernel). A present digest with no memo link (seeded into
    the tier) turns the witness off until it leaves; clears and evictions keep
    W exact. Every hit length equals the host index's LPM."""
    from paper_2510_09665_b200.api import Engine
    rng = np.random.default_rng(21)
    e = Engine(num_layers=2, bpt=64, page_tokens=16, tag=TAG, chunk_size=256, ram_slots=8, num_pages=4096)

    def lpm(p):
        keys = C.chunk_keys(p, 256, TAG)
        k = 0
        while k < len(keys) and e.contains(keys[k]):
            k += 1
        return min(len(p) - 1, 256 * k) if len(p) else 0

    qid = [100]

    def lookup(p):
        qid[0] += 1
        m = e.get_num_new_matched_tokens(qid[0], p)
        e.finish_query(qid[0])
        assert m == lpm(p)
        return m

    def store(p):
        qid[0] += 1
        q = qid[0]
        e.get_num_new_matched_tokens(q, p)
        e.bind_pages(q, len(p))
        e.update_state_after_alloc(q, (len(p) + 15) // 16, 0)
        m = e.build_connector_meta([(q, p)])
        S.transfer(e, m, q, p)
        e.drop_meta(m)
        e.finish_query(q)
        e.release_query(q)

    doc = rng.integers(0, 128256, size=256 * 4, dtype=np.uint32)
    store(doc)                                             # 4 chunks, linked by the planning hash
    w0 = e.lookups_witnessed()
    assert lookup(rng.integers(0, 128256, size=700, dtype=np.uint32)) == 0   # cold: first row witnessed
    assert e.lookups_witnessed() == w0 + 1
    q = np.concatenate([doc, rng.integers(0, 128256, size=60, dtype=np.uint32)])
    assert lookup(q) == 1024                               # stored doc + question: question row witnessed
    assert e.lookups_witnessed() == w0 + 2
    fork = np.concatenate([doc[:512], rng.integers(0, 128256, size=300, dtype=np.uint32)])
    assert lookup(fork) == 512                             # diverges inside chunk 2
    assert e.lookups_witnessed() == w0 + 3
    # a present digest without a link: the witness is off, results unchanged
    seeded = rng.integers(0, 128256, size=256 * 2, dtype=np.uint32)
    e.seed_store(seeded, 512)
    w1 = e.lookups_witnessed()
    assert lookup(rng.integers(0, 128256, size=400, dtype=np.uint32)) == 0
    assert lookup(q) == 1024
    assert lookup(seeded) == 511
    assert e.lookups_witnessed() == w1
    for k in C.chunk_keys(seeded, 256, TAG):               # they leave: the witness is back
        assert e.store_clear(k) == 1
    assert lookup(rng.integers(0, 128256, size=400, dtype=np.uint32)) == 0
    assert e.lookups_witnessed() == w1 + 1
    # evictions: the tier holds 8 chunks; two more documents push doc out
    for _ in range(2):
        store(rng.integers(0, 128256, size=256 * 3, dtype=np.uint32))
    lookup(q)
    lookup(doc)
    lookup(fork)
    assert e.store_clear(C.chunk_keys(doc, 256, TAG)[0]) in (0, 1)
    lookup(q)
    e.close()


def test_absence_witness_random_trace(tkv, C):
    """Random stores (through the connector), seeds without links, clears
    and evictions interleaved with lookups of prefixes, forks and fresh
    prompts: every hit length equals the host index's LPM, and the witness
    decides a good share of the absent rows."""
    from paper_2510_09665_b200.api import Engine
    rng = np.random.default_rng(5)
    e = Engine(num_layers=1, bpt=32, page_tokens=16, tag=TAG, chunk_size=256, ram_slots=24, num_pages=8192)
    docs, qid = [], [0]

    def lpm(p):
        keys = C.chunk_keys(p, 256, TAG)
        k = 0
        while k < len(keys) and e.contains(keys[k]):
            k += 1
        return min(len(p) - 1, 256 * k) if len(p) else 0

    def next_q():
        qid[0] += 1
        return qid[0]

    seeded = []
    for step in range(160):
        op = rng.random()
        if op < 0.25 or not docs:
            p = rng.integers(0, 128256, size=int(rng.integers(1, 6)) * 256 + int(rng.integers(0, 200)), dtype=np.uint32)
            q = next_q()
            e.get_num_new_matched_tokens(q, p)
            e.bind_pages(q, len(p))
            e.update_state_after_alloc(q, (len(p) + 15) // 16, 0)
            m = e.build_connector_meta([(q, p)])
            S.transfer(e, m, q, p)
            e.drop_meta(m)
            e.finish_query(q)
            e.release_query(q)
            docs.append(p)
        elif op < 0.30:
            p = rng.integers(0, 128256, size=256 * int(rng.integers(1, 3)), dtype=np.uint32)
            e.seed_store(p, len(p))
            seeded.append(p)
        elif op < 0.38 and seeded:
            p = seeded.pop(int(rng.integers(0, len(seeded))))
            for k in C.chunk_keys(p, 256, TAG):
                e.store_clear(k)
        elif op < 0.42:
            d = docs[int(rng.integers(0, len(docs)))]
            for k in C.chunk_keys(d, 256, TAG)[int(rng.integers(0, 3)):]:
                e.store_clear(k)
        else:
            d = docs[int(rng.integers(0, len(docs)))]
            r = rng.random()
            if r < 0.4:
                p = np.concatenate([d, rng.integers(0, 128256, size=int(rng.integers(1, 100)), dtype=np.uint32)])
            elif r < 0.7:
                cut = int(rng.integers(1, len(d) + 1))
                p = np.concatenate([d[:cut], rng.integers(0, 128256, size=int(rng.integers(1, 400)), dtype=np.uint32)])
            else:
                p = rng.integers(0, 128256, size=int(rng.integers(1, 1500)), dtype=np.uint32)
            q = next_q()
            assert e.get_num_new_matched_tokens(q, p) == lpm(p), step
            e.finish_query(q)
    assert e.lookups_witnessed() > 10
    e.close()
