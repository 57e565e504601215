"""Config-4 lookup latency, B200 connector vs the reference Connector, on the
same prompts (get_num_new_matched_tokens through each C-ABI / shim):

  hit   a stored 128K-token document + a 60-token question: the reference
        hashes every chunk up to the first absent one (the question), so 513
        SHA-256 chunks; the B200 path probes the prefix memo (warm after the
        first lookup) and hashes the one new chunk.
  miss  a cold 128K-token document: both stop at the first chunk.

The lookup does not depend on the KV geometry, so both engines use one layer
of 64-byte rows (the stored chunks' bytes are irrelevant to the lookup).
The B200 tier gets the document the way config 4 does: a cold prefill stored
through the connector (its planning hash links every chunk, so the absence
witness is on); `--seeded` puts it straight into the tier instead (no links:
the witness stays off and every absent row is hashed). One JSON line."""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
from paper_2510_09665_b200.api import Engine  # noqa: E402

TAG, N_DOC = "llama-3.1-8b", 131072
GEOM = dict(num_layers=1, bpt=64, page_tokens=16, tag=TAG, chunk_size=256, ram_slots=N_DOC // 256 + 8,
            num_pages=64)


def toks(n, seed):
    return np.random.default_rng(seed).integers(0, 128256, size=n, dtype=np.uint32)


def timed_lookups(e, prompts, qid0, prepare=None):
    ts = []
    for i, p in enumerate(prompts):
        if prepare:
            prepare(qid0 + i, p)
        t0 = time.perf_counter()
        m = e.get_num_new_matched_tokens(qid0 + i, p)
        ts.append(time.perf_counter() - t0)
        e.finish_query(qid0 + i)
    return ts, m


def store_through_connector(e, qid, p):
    """A cold prefill of p stored by the connector (layerwise store)."""
    e.get_num_new_matched_tokens(qid, p)
    e.bind_pages(qid, len(p))
    e.update_state_after_alloc(qid, (len(p) + 15) // 16, 0)
    m = e.build_connector_meta([(qid, p)])
    assert e.start_load_kv(m) == 0
    e.compute_range(qid, p, 0, len(p), layers=(0, 1))
    assert e.start_store_kv(m) == 0
    if e.meta_layerwise(m):
        assert e.wait_store_kv(m, 0) == 0
    e.synchronize()
    e.drop_meta(m)
    e.finish_query(qid)
    e.release_query(qid)


def main(reps=20, seeded=False):
    doc = toks(N_DOC, 5)
    hits = [np.concatenate([doc, toks(60, 100 + i)]) for i in range(reps + 1)]
    misses = [toks(N_DOC, 1000 + i) for i in range(reps)]
    e = Engine(**dict(GEOM, num_pages=N_DOC // 16 + 64))
    if seeded:
        e.seed_store(doc, N_DOC)
    else:
        store_through_connector(e, 99999, doc)
    prep = (lambda q, p: (e.dev_prompt(q, p), torch.cuda.synchronize()))
    t_first, _ = timed_lookups(e, hits[:1], 1, prep)  # memo cold: every chunk through SHA
    t_hit, m_hit = timed_lookups(e, hits[1:], 100, prep)
    t_miss, m_miss = timed_lookups(e, misses, 1000, prep)
    assert m_hit == N_DOC and m_miss == 0
    out = {"lookup": "c4: 128K-token document (+ 60-token question)", "tokens_hit": len(hits[0]),
           "b200_hit_first_ms": round(1e3 * t_first[0], 3),
           "b200_hit_ms_median": round(1e3 * float(np.median(t_hit)), 3),
           "b200_miss_ms_median": round(1e3 * float(np.median(t_miss)), 3), "memo": e.memo_stats(),
           "tier": "seeded (no memo links)" if seeded else "stored through the connector",
           "witnessed_rows": e.lookups_witnessed()}
    e.close()
    if oracle.ref_available():
        r = oracle.RefEngine(**GEOM)
        r.seed_store(doc, N_DOC)
        rh, rm_hit = timed_lookups(r, hits[:5], 1)
        rm, rm_miss = timed_lookups(r, misses[:5], 100)
        assert rm_hit == N_DOC and rm_miss == 0
        out.update({"ref_hit_ms_median": round(1e3 * float(np.median(rh)), 3),
                    "ref_miss_ms_median": round(1e3 * float(np.median(rm)), 3), "ref_cores": 1})
        r.close()
    print(json.dumps(out))


if __name__ == "__main__":
    main(seeded="--seeded" in sys.argv)
