"""Generates the golden fixtures in tests/golden/ from the UNMODIFIED reference
(oracle/_ref/libtierkv_ref.so, compiled from /root/reference/proj/src by
oracle/Makefile). Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

Fixtures:
  keys.json       chunk_keys digests for fixed and seeded token sequences,
                  several chunk sizes and tag lengths (tokens.cpp:49-57);
                  LPM results against stored digest sets (tokens.cpp:59-69)
  synth.json      sha256 / fnv1a64 of synth_layer_kv slabs (synth.cpp:22-30)
  scenarios.json  observable outcomes of tests/scenarios.py run on the
                  reference engine (Connector/TieredStore/PagedKVStore)
"""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))

import oracle  # noqa: E402
import scenarios as S  # noqa: E402


def key_cases():
    cases = [("range600", list(range(600)), 256, "m"),
             ("mul7919", [(i * 7919) % 128256 for i in range(1000)], 256, "llama-3.1-8b")]
    rng = np.random.default_rng(2510)
    for cs in (1, 16, 256, 257):
        for n in (0, 1, 255, 256, 257, 1000, 4096):
            if cs == 1 and n > 300:
                continue
            cases.append((f"rand_cs{cs}_n{n}", rng.integers(0, 128256, size=n).tolist(), cs, "llama-3.1-8b"))
    for tl in (0, 1, 29, 30, 40, 200):
        cases.append((f"tag{tl}", rng.integers(0, 128256, size=700).tolist(), 256, "t" * tl))
    return cases


def main():
    R = oracle.Ref()
    keys = []
    for name, toks, cs, tag in key_cases():
        keys.append({"name": name, "tokens": toks, "chunk_size": cs, "tag": tag,
                     "digests": [d.hex() for d in R.chunk_keys(toks, cs, tag)]})
    lpm = []
    rng = np.random.default_rng(99)
    for i in range(12):
        q = rng.integers(0, 32000, size=int(rng.integers(1, 3000))).tolist()
        keep = int(rng.integers(0, len(q) + 1))
        stored = R.chunk_keys(q[:keep], 256, "m")
        lpm.append({"tokens": q, "stored": [d.hex() for d in stored],
                    "match": R.longest_prefix_match(q, 256, "m", stored)})
    seed = R.model_seed("llama-3.1-8b")
    synth = []
    t = [(i * 7919) % 128256 for i in range(1000)]
    for layer, bpt, first in [(5, 4096, 0), (0, 512, 256), (79, 512, 768), (3, 64, 10)]:
        slab = R.synth_layer_kv(seed, t[first:first + 256], layer, first, bpt)
        synth.append({"layer": layer, "bpt": bpt, "first_pos": first, "tag": "llama-3.1-8b",
                      "sha256": hashlib.sha256(slab.tobytes()).hexdigest(), "fnv1a64": R.fnv1a64(slab)})
    out = {"model_seed": {"llama-3.1-8b": seed}, "model_tag_hash": {"llama-3.1-8b": R.model_tag_hash("llama-3.1-8b")}}
    with open(os.path.join(HERE, "keys.json"), "w") as f:
        json.dump({"keys": keys, "lpm": lpm, **out}, f)
    with open(os.path.join(HERE, "synth.json"), "w") as f:
        json.dump({"tokens": t, "slabs": synth, **out}, f, indent=1)
    q8 = []
    rng = np.random.default_rng(8)
    for n in (2, 3, 100, 4096, 4097, 70000):
        p = rng.integers(0, 256, size=n, dtype=np.uint8)
        blob = R.q8_encode(p)
        dec, code = R.q8_decode(blob)
        q8.append({"seed": 8, "n": n, "blob_sha256": hashlib.sha256(blob.tobytes()).hexdigest(),
                   "decoded_sha256": hashlib.sha256(dec.tobytes()).hexdigest()})
    with open(os.path.join(HERE, "q8.json"), "w") as f:
        json.dump({"note": "payloads: np.random.default_rng(8).integers(0, 256, size=n) in order", "cases": q8},
                  f, indent=1)
    C = oracle.C()
    sc = {fn.__name__: json.loads(json.dumps(fn(S.ref_factory, C))) for fn in S.ALL}
    with open(os.path.join(HERE, "scenarios.json"), "w") as f:
        json.dump(sc, f, indent=1)
    print("wrote keys.json synth.json scenarios.json")


if __name__ == "__main__":
    main()
