"""Full-size parity at the BASELINE.json configs' shapes, through the C-ABI
connector: store a cold prompt, retrieve it into fresh pages, and check
(1) every stored chunk payload against the CPU oracle (checksum of each
chunk, all chunks), (2) every retrieved page on device against the synth
oracle (K4 verifier), (3) random rows against the CPU oracle byte for byte.
The oracle here is the reference's own engine byte oracle, synth_layer_kv
recomputation (sim_engine.cpp:66-81, 474-490)."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _cold_then_warm(e, prompt, qid_cold, qid_warm):
    n, L = len(prompt), e.num_layers
    assert e.get_num_new_matched_tokens(qid_cold, prompt) == 0
    e.bind_pages(qid_cold, n)
    e.update_state_after_alloc(qid_cold, (n + 15) // 16, 0)
    m = e.build_connector_meta([(qid_cold, prompt)])
    assert e.start_load_kv(m) == 0
    for layer in range(L):
        e.wait_load_kv(m, layer)
        e.compute_range(qid_cold, prompt, 0, n, layers=(layer, layer + 1))
        if layer:
            assert e.wait_store_kv(m, layer - 1) == 0
        assert e.start_store_kv(m) == 0
    assert e.wait_store_kv(m, L - 1) == 0
    res = e.store_results(m, qid_cold)
    assert all(c == 0 for _, c in res)
    e.finish_query(qid_cold)
    e.release_query(qid_cold)
    assert e.get_num_new_matched_tokens(qid_warm, prompt) == n - 1
    e.bind_pages(qid_warm, n)
    e.update_state_after_alloc(qid_warm, (n + 15) // 16, (n - 1 + 15) // 16)
    m2 = e.build_connector_meta([(qid_warm, prompt)])
    assert e.start_load_kv(m2) == 0
    for layer in range(L):
        e.wait_load_kv(m2, layer)
    e.synchronize()
    assert e.loaded_tokens(m2, qid_warm) == n - 1
    return [d for d, _ in res]


def test_config1_shape_store_retrieve(tkv, C):
    """8B: 32 layers x 4096 B/token-layer, 4096-token prompt (512 MiB)."""
    from paper_2510_09665_b200.api import Engine
    tag, L, bpt, n = "llama-3.1-8b", 32, 4096, 4096
    rng = np.random.default_rng(1)
    prompt = rng.integers(0, 128256, size=n, dtype=np.uint32)
    e = Engine(num_layers=L, bpt=bpt, page_tokens=16, tag=tag, chunk_size=256, ram_slots=17,
               num_pages=2 * L * n // 16 + 64, staging_budget=1 << 32)
    digests = _cold_then_warm(e, prompt, 1, 2)
    assert digests == C.chunk_keys(prompt, 256, tag)
    seed = C.model_seed(tag)
    for i, d in enumerate(digests):
        got = e.store_get(d)
        want = C.synth_chunk(seed, prompt, 256 * i, 256, L, bpt)
        assert C.fnv1a64(got) == C.fnv1a64(want), f"chunk {i}"
    assert e.verify_range(2, prompt, 0, n - 1) == 0
    for _ in range(8):
        layer, tok = int(rng.integers(0, L)), int(rng.integers(0, n - 1))
        row = e.gather_layer(2, layer, tok + 1)[tok * bpt:(tok + 1) * bpt]
        assert np.array_equal(row, C.synth_token_kv(seed, int(prompt[tok]), layer, tok, bpt))
    e.close()


@pytest.mark.parametrize("tp", [8, 2])
def test_config3_shape_tp_shard(tkv, C, tp):
    """70B at TP=tp: 80 layers, bpt 4096/tp, 8K-token prompt per rank shard."""
    from paper_2510_09665_b200.api import Engine
    tag, L, bpt, n = "llama-3.1-70b", 80, 4096 // tp, 8192
    rng = np.random.default_rng(tp)
    prompt = rng.integers(0, 128256, size=n, dtype=np.uint32)
    e = Engine(num_layers=L, bpt=bpt, page_tokens=16, tag=tag, chunk_size=256, ram_slots=33,
               num_pages=2 * L * n // 16 + 64, staging_budget=1 << 32)
    digests = _cold_then_warm(e, prompt, 1, 2)
    assert e.verify_range(2, prompt, 0, n - 1) == 0
    seed = C.model_seed(tag)
    for i in (0, len(digests) - 1):
        assert np.array_equal(e.store_get(digests[i]), C.synth_chunk(seed, prompt, 256 * i, 256, L, bpt))
    e.close()
