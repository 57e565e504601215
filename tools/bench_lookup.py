"""Config-4 lookup latency: get_num_new_matched_tokens of a 128K-token
document + question through the C-ABI connector, memo cold (first lookup:
SHA of every chunk) and warm (every chunk a memo hit), vs the reference's own
chunk_keys (oracle/_ref, OpenSSL SHA-NI, one core). One JSON line."""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2510_09665_b200.api import Engine  # noqa: E402


def main():
    n_doc, reps = 131072, 20
    rng = np.random.default_rng(5)
    doc = rng.integers(0, 128256, size=n_doc, dtype=np.uint32)
    e = Engine(num_layers=32, bpt=4096, page_tokens=16, tag="llama-3.1-8b", chunk_size=256,
               ram_slots=4, num_pages=256)
    prompts = [np.concatenate([doc, rng.integers(0, 128256, size=60, dtype=np.uint32)]) for _ in range(reps + 1)]
    e.dev_prompt(1, prompts[0])
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e.get_num_new_matched_tokens(1, prompts[0])
    cold = time.perf_counter() - t0
    warm = []
    for i in range(reps):
        e.dev_prompt(2 + i, prompts[1 + i])  # the engine's own prompt upload, not part of the lookup
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e.get_num_new_matched_tokens(2 + i, prompts[1 + i])
        warm.append(time.perf_counter() - t0)
        e.finish_query(2 + i)
        e.release_query(2 + i)
    st = e.memo_stats()
    e.close()
    ref = None
    import oracle
    if oracle.ref_available():
        R = oracle.Ref()
        ts = []
        for _ in range(5):
            t0 = time.perf_counter()
            R.chunk_keys(prompts[0], 256, "llama-3.1-8b")
            ts.append(time.perf_counter() - t0)
        ref = round(1e3 * min(ts), 3)
    print(json.dumps({"lookup": "c4 128K doc + 60-token question", "tokens": len(prompts[0]),
                      "cold_ms": round(1e3 * cold, 3), "warm_ms_median": round(1e3 * float(np.median(warm)), 3),
                      "warm_ms_min": round(1e3 * min(warm), 3), "memo": st, "ref_cpu_chunk_keys_ms_1core": ref}))


if __name__ == "__main__":
    main()
