"""CPU: pins the oracle (oracle/tierkv_oracle.c) before anything is checked
against it — SURVEY.md Appendix A vectors, the reference-generated fixtures
in tests/golden/, and (where oracle/_ref exists) the reference itself on
seeded random inputs."""
import hashlib
import json
import os

import numpy as np
import pytest

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def test_appendix_a_keys(C):
    assert [k.hex() for k in C.chunk_keys(list(range(600)), 256, "m")] == [
        "5adb258b77fe3a6f5d2341135db04896c6bd5d5e13bb18923c88e5247cef9dc0",
        "c153731d406774e9d83ac9fbad6414e6ffa2c838afd908b48a3701230faac9b3",
        "7764a4adf62fa1e539afebddb8905ff5457aee5ce4c234d036cc8dd90a0376d4"]
    t = [(i * 7919) % 128256 for i in range(1000)]
    assert [k.hex() for k in C.chunk_keys(t, 256, "llama-3.1-8b")] == [
        "4ac68da485c720853487c36c92e79af957b3bfb514b4cd0a8c1a75d28e574831",
        "e67ecd2e864d42958ce0f1e3a5da5e69ddb87e47b57c76fbf63579f5417516d7",
        "39da76fef676a9ed6f0f7a91db987bbe60dde3c0fcd477ef80059af788910a9e",
        "b051f7c6957dd2d1db868787f5054fab9a067435807a75ef271bd34f941884e2"]


def test_appendix_a_seeds_and_synth(C):
    assert C.model_seed("llama-3.1-8b") == 0x67891337732B2A04
    assert C.model_tag_hash("llama-3.1-8b") == 0xD3D294D00935637B
    seed = C.model_seed("llama-3.1-8b")
    assert C.synth_token_kv(seed, 42, 3, 100, 16).tobytes().hex() == "be717690e0643389d6c054fed16083da"
    t = [(i * 7919) % 128256 for i in range(256)]
    slab = C.synth_layer_kv(seed, t, 5, 0, 4096)
    assert hashlib.sha256(slab.tobytes()).hexdigest() == \
        "d365ad9a1d63eb66b01ee65c9794133b584a68102ea4666c60ce6de69d252109"
    assert C.fnv1a64(slab) == 0x938297F9C3A70E30


def test_sha256_fips_vectors(C):
    assert C.sha256(b"").hex() == "e3b0c44298fc1c149afbf4c8996fb92427ae41e4649b934ca495991b7852b855"
    assert C.sha256(b"abc").hex() == "ba7816bf8f01cfea414140de5dae2223b00361a396177a9cb410ff61f20015ad"
    msg = b"abcdbcdecdefdefgefghfghighijhijkijkljklmklmnlmnomnopnopq"
    assert C.sha256(msg).hex() == "248d6a61d20638b8e5c026930c3e6039a33ce45964ff2167f6ecedd419db06c1"
    for n in (55, 56, 63, 64, 65, 1070):
        data = bytes(range(256)) * 5
        assert C.sha256(data[:n]) == hashlib.sha256(data[:n]).digest()


def test_golden_keys(C):
    with open(os.path.join(GOLDEN, "keys.json")) as f:
        g = json.load(f)
    for case in g["keys"]:
        got = [d.hex() for d in C.chunk_keys(case["tokens"], case["chunk_size"], case["tag"])]
        assert got == case["digests"], case["name"]
    for case in g["lpm"]:
        stored = [bytes.fromhex(d) for d in case["stored"]]
        assert C.longest_prefix_match(case["tokens"], 256, "m", stored) == case["match"]
    assert C.model_seed("llama-3.1-8b") == g["model_seed"]["llama-3.1-8b"]
    assert C.model_tag_hash("llama-3.1-8b") == g["model_tag_hash"]["llama-3.1-8b"]


def test_golden_synth(C):
    with open(os.path.join(GOLDEN, "synth.json")) as f:
        g = json.load(f)
    seed = C.model_seed("llama-3.1-8b")
    t = g["tokens"]
    for s in g["slabs"]:
        slab = C.synth_layer_kv(seed, t[s["first_pos"]:s["first_pos"] + 256], s["layer"], s["first_pos"], s["bpt"])
        assert hashlib.sha256(slab.tobytes()).hexdigest() == s["sha256"]
        assert C.fnv1a64(slab) == s["fnv1a64"]


def test_gather_scatter_restatement(C):
    """paged_store.cpp:123-175: scatter then gather is the identity, the final
    page takes only n mod page_tokens rows."""
    rng = np.random.default_rng(1)
    bpt, pt = 64, 16
    pool = np.zeros(32 * pt * bpt, np.uint8)
    for n in (1, 16, 33, 48, 255):
        pages = rng.permutation(32)[: (n + pt - 1) // pt]
        data = rng.integers(0, 256, size=n * bpt, dtype=np.uint8)
        C.scatter_tokens(pool, pt * bpt, pages, bpt, n, data)
        assert np.array_equal(C.gather_tokens(pool, pt * bpt, pages, bpt, n), data)


def test_oracle_equals_reference_random(C, Ref):
    rng = np.random.default_rng(123)
    for _ in range(40):
        n = int(rng.integers(0, 2000))
        cs = int(rng.choice([1, 7, 16, 256, 257]))
        tag = "x" * int(rng.integers(0, 60))
        t = rng.integers(0, 2**32, size=n, dtype=np.uint64).astype(np.uint32)
        assert C.chunk_keys(t, cs, tag) == Ref.chunk_keys(t, cs, tag)
    seed = Ref.model_seed("conn-test")
    for bpt in (8, 12, 64, 4096):
        t = rng.integers(0, 32000, size=50).astype(np.uint32)
        assert np.array_equal(C.synth_layer_kv(seed, t, 3, 77, bpt), Ref.synth_layer_kv(seed, t, 3, 77, bpt))


def test_lpm_brute_force(C):
    """test_tokens.cpp:193-223: LPM equals the brute-force prefix oracle."""
    rng = np.random.default_rng(16)

    def brute(q, stored, cs):
        best = 0
        for s in stored:
            p = 0
            while p < min(len(q), len(s)) and q[p] == s[p]:
                p += 1
            m = p if (p == len(q) and len(s) == len(q)) else (p // cs) * cs
            best = max(best, m)
        return best

    for it in range(20):
        cs = 16 if it % 2 == 0 else 7
        base = rng.integers(0, 32000, size=200).tolist()
        stored = []
        for _ in range(5):
            keep = int(rng.integers(0, 201))
            stored.append(base[:keep] + rng.integers(0, 32000, size=int(rng.integers(0, 201))).tolist())
        digests = [d for s in stored for d in C.chunk_keys(s, cs, "m")]
        for qn in range(6):
            q = base[:int(rng.integers(0, 201))] + rng.integers(0, 32000, size=int(rng.integers(0, 40))).tolist()
            if qn == 5:
                q = stored[0]
            assert C.longest_prefix_match(q, cs, "m", digests) == brute(q, stored, cs)


@pytest.mark.parametrize("name", ["keys", "scenarios"])
def test_fixtures_regenerate_identically(Ref, name):
    """The committed fixtures are exactly what the reference produces now."""
    import sys
    sys.path.insert(0, os.path.dirname(__file__))
    import oracle
    import scenarios as S
    if name == "scenarios":
        with open(os.path.join(GOLDEN, "scenarios.json")) as f:
            g = json.load(f)
        C = oracle.C()
        for fn in S.ALL:
            assert json.loads(json.dumps(fn(S.ref_factory, C))) == g[fn.__name__], fn.__name__
    else:
        with open(os.path.join(GOLDEN, "keys.json")) as f:
            g = json.load(f)
        for case in g["keys"][:10]:
            got = [d.hex() for d in Ref.chunk_keys(case["tokens"], case["chunk_size"], case["tag"])]
            assert got == case["digests"]
