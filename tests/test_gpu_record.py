"""LMCK record framing (chunk_file.cpp): a chunk
exported from the pinned tier is byte-identical to the reference's
encode_chunk_record of the same chunk; a reference record imports into the
tier; corruption / truncation / trailing bytes give corrupt_chunk and a
foreign geometry gives invalid_argument (test_formats.cpp:25-96)."""
import ctypes as ct

import numpy as np
import pytest

import scenarios as S

pytestmark = pytest.mark.gpu

TAG = "fmt-test"


def _tag_hash(lib, tag):
    v = ct.c_uint64(0)
    assert lib.tkv_model_tag_hash(tag.encode(), ct.byref(v)) == 0
    return v.value


def test_model_tag_hash_on_device(tkv, C):
    lib = tkv.lib()
    for tag in ("fmt-test", "llama-3.1-8b", "", "x" * 200):
        assert _tag_hash(lib, tag) == C.model_tag_hash(tag)


def test_export_matches_reference_and_import_roundtrip(tkv, C, Ref):
    from paper_2510_09665_b200._lib import u8p
    from paper_2510_09665_b200.api import Engine
    lib = tkv.lib()
    e = Engine(num_layers=4, bpt=64, page_tokens=16, tag=TAG, chunk_size=32, ram_slots=8, num_pages=64)
    prompt = S.make_prompt(70, 3)  # chunks of 32, 32, 6 tokens
    e.seed_store(prompt, 70)
    keys = C.chunk_keys(prompt, 32, TAG)
    th = _tag_hash(lib, TAG)
    seed = C.model_seed(TAG)
    records = []
    for i, k in enumerate(keys):
        n_tok = min(32, 70 - 32 * i)
        d = np.frombuffer(k, np.uint8).copy()
        n = ct.c_size_t(0)
        assert lib.tkv_store_export_record(e.store, d.ctypes.data_as(u8p), th, None, 0, ct.byref(n)) == 0
        out = np.zeros(n.value, np.uint8)
        assert lib.tkv_store_export_record(e.store, d.ctypes.data_as(u8p), th, out.ctypes.data_as(u8p),
                                           out.size, ct.byref(n)) == 0
        payload = C.synth_chunk(seed, prompt, 32 * i, n_tok, 4, 64)
        want = Ref.encode_record(TAG, k, n_tok, 4, 64, payload)
        assert np.array_equal(out, want), i
        code, back = Ref.parse_record(out, payload.size)
        assert code == 0 and np.array_equal(back, payload)
        records.append((k, want, payload))
    e.close()

    f = Engine(num_layers=4, bpt=64, page_tokens=16, tag=TAG, chunk_size=32, ram_slots=8, num_pages=64)
    for k, rec, payload in records:
        assert lib.tkv_store_import_record(f.store, rec.ctypes.data_as(u8p), rec.size, 0) == 0
        assert np.array_equal(f.store_get(k), payload)
    rec = records[0][1]
    bad = rec.copy()
    bad[0] = ord("X")
    assert lib.tkv_store_import_record(f.store, bad.ctypes.data_as(u8p), bad.size, 0) == 5
    bad = rec.copy()
    bad[4] = 9
    assert lib.tkv_store_import_record(f.store, bad.ctypes.data_as(u8p), bad.size, 0) == 5
    bad = rec.copy()
    bad[54 + 5] ^= 0x40  # header is 54 bytes (chunk_file.hpp:18)
    assert lib.tkv_store_import_record(f.store, bad.ctypes.data_as(u8p), bad.size, 0) == 5
    for keep in (0, 3, 53, 54, rec.size - 9, rec.size - 1):
        t = rec[:keep].copy()
        assert lib.tkv_store_import_record(f.store, t.ctypes.data_as(u8p), t.size, 0) == 5
    longer = np.concatenate([rec, np.zeros(1, np.uint8)])
    assert lib.tkv_store_import_record(f.store, longer.ctypes.data_as(u8p), longer.size, 0) == 5
    f.close()
    g = Engine(num_layers=2, bpt=64, page_tokens=16, tag=TAG, chunk_size=32, ram_slots=8, num_pages=64)
    assert lib.tkv_store_import_record(g.store, rec.ctypes.data_as(u8p), rec.size, 0) == 16
    g.close()


def test_record_bit_flips_match_reference_parse(tkv, C, Ref):
    """Every single-bit flip of the header, the trailing checksum and sampled
    payload bytes: import into the tier fails exactly when the reference's
    parse_chunk_record (chunk_file.cpp:47-95) rejects the record, with the
    same Errc; an accepted record stores the payload the reference parsed."""
    from paper_2510_09665_b200._lib import u8p
    from paper_2510_09665_b200.api import Engine
    lib = tkv.lib()
    prompt = S.make_prompt(40, 9)
    keys = C.chunk_keys(prompt, 32, TAG)
    payload = C.synth_chunk(C.model_seed(TAG), prompt, 32, 8, 4, 64)  # the 8-token tail chunk
    rec = Ref.encode_record(TAG, keys[1], 8, 4, 64, payload)
    rng = np.random.default_rng(5)
    positions = list(range(54)) + list(range(rec.size - 8, rec.size)) + \
        sorted(rng.choice(np.arange(54, rec.size - 8), 40, replace=False).tolist())
    e = Engine(num_layers=4, bpt=64, page_tokens=16, tag=TAG, chunk_size=32, ram_slots=4, num_pages=64)
    accepted = 0
    for pos in positions:
        for bit in (0, 3, 7):
            bad = rec.copy()
            bad[pos] ^= np.uint8(1 << bit)
            want, back = Ref.parse_record(bad, payload.size)
            got = lib.tkv_store_import_record(e.store, bad.ctypes.data_as(u8p), bad.size, 0)
            assert got == want, (pos, bit, got, want)
            if got == 0:  # accepted: stored under the record's digest, bytes as parsed
                dig = np.zeros(32, np.uint8)
                geo = (ct.c_uint32 * 3)()
                th = ct.c_uint64(0)
                assert lib.tkv_record_peek(bad.ctypes.data_as(u8p), bad.size, dig.ctypes.data_as(u8p), geo,
                                           ct.byref(th)) == 0
                assert np.array_equal(e.store_get(dig.tobytes()), back)
                e.store_clear(dig.tobytes())
                accepted += 1
    e.close()
