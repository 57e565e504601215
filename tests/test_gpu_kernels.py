"""Kernel parity on the B200: K3 (chained SHA-256 keys), K1/K2 (paged
gather/scatter), K4 (synthetic KV) against the CPU oracle (oracle/), byte for
byte. Shapes cover the reference tests' edge cases (empty, ragged tails,
chunk sizes 1/16/256/257, tag lengths that push the parent digest across a
SHA block boundary) and the configs' geometries (bpt 4096 / 512)."""
import ctypes as ct
import random

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def rand_tokens(rng, n, vocab=128256):
    return rng.integers(0, vocab, size=n, dtype=np.uint32)


# ---------------------------------------------------------------- K3 -------

def test_keys_appendix_a(tkv):
    from paper_2510_09665_b200.api import chunk_keys
    got = [k.hex() for k in chunk_keys(list(range(600)), 256, "m")]
    assert got == ["5adb258b77fe3a6f5d2341135db04896c6bd5d5e13bb18923c88e5247cef9dc0",
                   "c153731d406774e9d83ac9fbad6414e6ffa2c838afd908b48a3701230faac9b3",
                   "7764a4adf62fa1e539afebddb8905ff5457aee5ce4c234d036cc8dd90a0376d4"]
    t2 = [(i * 7919) % 128256 for i in range(1000)]
    got = [k.hex() for k in chunk_keys(t2, 256, "llama-3.1-8b")]
    assert got == ["4ac68da485c720853487c36c92e79af957b3bfb514b4cd0a8c1a75d28e574831",
                   "e67ecd2e864d42958ce0f1e3a5da5e69ddb87e47b57c76fbf63579f5417516d7",
                   "39da76fef676a9ed6f0f7a91db987bbe60dde3c0fcd477ef80059af788910a9e",
                   "b051f7c6957dd2d1db868787f5054fab9a067435807a75ef271bd34f941884e2"]


@pytest.mark.parametrize("cs", [1, 16, 256, 257])
def test_keys_match_oracle_random(tkv, C, cs):
    from paper_2510_09665_b200.api import chunk_keys
    rng = np.random.default_rng(cs)
    for n in [0, 1, cs - 1 if cs > 1 else 2, cs, cs + 1, 3 * cs + 7, 1000]:
        t = rand_tokens(rng, n)
        assert chunk_keys(t, cs, "m") == C.chunk_keys(t, cs, "m"), (cs, n)


@pytest.mark.parametrize("tag", ["", "m", "llama-3.1-8b", "x" * 29, "y" * 30, "z" * 40, "t" * 200])
def test_keys_tag_lengths(tkv, C, tag):
    """Tag length moves the parent digest and the token stream across SHA
    block boundaries and changes the token byte misalignment."""
    from paper_2510_09665_b200.api import chunk_keys
    rng = np.random.default_rng(len(tag))
    for n in [1, 5, 255, 256, 600]:
        t = rand_tokens(rng, n)
        assert chunk_keys(t, 256, tag) == C.chunk_keys(t, 256, tag), (len(tag), n)


def test_keychain_resume(tkv, C):
    from paper_2510_09665_b200.api import chunk_keys, keychain_next
    rng = np.random.default_rng(14)
    t = rand_tokens(rng, 700)
    direct = chunk_keys(t, 256, "m")
    assert keychain_next("m", 256, direct[1], t[512:700]) == direct[2]


def test_hash_chains_many_requests(tkv, C):
    """One launch over many independent chains of ragged lengths (K3 over
    requests), checked chain by chain against the oracle."""
    from paper_2510_09665_b200.api import ChainDescC, hash_chains
    rng = np.random.default_rng(7)
    lens = [int(x) for x in rng.integers(0, 3000, size=97)] + [0, 1, 256, 4096]
    toks = [rand_tokens(rng, n) for n in lens]
    flat = np.concatenate(toks + [np.zeros(1, np.uint32)])
    chains = (ChainDescC * len(lens))()
    off = row = 0
    for i, n in enumerate(lens):
        chains[i].token_off = off
        chains[i].n_tokens = n
        chains[i].out_first = row
        off += n
        row += (n + 255) // 256
    dev_t = torch.from_numpy(flat.view(np.int32)).cuda()
    dev_c = torch.frombuffer(bytearray(bytes(chains)), dtype=torch.uint8).cuda()
    out = torch.zeros(max(1, row) * 32, dtype=torch.uint8, device="cuda")
    hash_chains(dev_t, dev_c, len(lens), 256, "llama-3.1-8b", out)
    torch.cuda.synchronize()
    o = out.cpu().numpy()
    row = 0
    for t in toks:
        want = C.chunk_keys(t, 256, "llama-3.1-8b")
        got = [o[32 * (row + i):32 * (row + i + 1)].tobytes() for i in range(len(want))]
        assert got == want
        row += len(want)


# ---------------------------------------------------------------- K4 -------

def test_synth_chunk_matches_oracle(tkv, C):
    from paper_2510_09665_b200._lib import check, lib
    rng = np.random.default_rng(3)
    seed = C.model_seed("llama-3.1-8b")
    for bpt, n, L in [(4096, 256, 3), (512, 100, 4), (64, 33, 2), (12, 17, 3), (8, 5, 1)]:
        prompt = rand_tokens(rng, 300)
        start = 16
        dev_t = torch.from_numpy(prompt.view(np.int32)).cuda()
        out = torch.zeros(L * n * bpt, dtype=torch.uint8, device="cuda")
        check(lib().tkv_synth_chunk(dev_t.data_ptr(), seed, start, n, L, bpt, out.data_ptr(), None))
        torch.cuda.synchronize()
        want = C.synth_chunk(seed, prompt, start, n, L, bpt)
        assert np.array_equal(out.cpu().numpy(), want), (bpt, n, L)


# ------------------------------------------------------------- K1/K2 -------

def _engine(tkv, L, bpt, pages, tag="k-test"):
    from paper_2510_09665_b200.api import Engine
    return Engine(num_layers=L, bpt=bpt, page_tokens=16, tag=tag, chunk_size=256, ram_slots=2,
                  num_pages=pages)


@pytest.mark.parametrize("bpt", [8, 64, 512, 4096])
def test_scatter_gather_roundtrip(tkv, bpt):
    """test_kv_core.cpp:136-156 — token counts {1,16,33,48,255} x 4 layers."""
    from paper_2510_09665_b200._lib import check, u8p, u32p
    e = _engine(tkv, 4, bpt, 64)
    rng = np.random.default_rng(21)
    for n in [1, 16, 33, 48, 255]:
        need = (n + 15) // 16
        ids = np.zeros(need, np.uint32)
        check(e.L.tkv_pages_alloc(e.pages, 7, need, ids.ctypes.data_as(u32p)))
        for layer in range(4):
            buf = rng.integers(0, 256, size=n * bpt, dtype=np.uint8)
            check(e.L.tkv_pages_scatter(e.pages, buf.ctypes.data_as(u8p), buf.size, ids.ctypes.data_as(u32p),
                                        ids.size, layer, n))
            back = np.zeros(n * bpt, np.uint8)
            check(e.L.tkv_pages_gather(e.pages, ids.ctypes.data_as(u32p), ids.size, layer, n,
                                       back.ctypes.data_as(u8p), back.size))
            assert np.array_equal(back, buf)
        e.L.tkv_pages_release(e.pages, 7)
    e.close()


def test_gather_checks(tkv):
    """test_kv_core.cpp:158-189 — unpopulated / wrong layer / size mismatch."""
    from paper_2510_09665_b200._lib import check, u8p, u32p
    e = _engine(tkv, 4, 64, 8)
    ids = np.zeros(2, np.uint32)
    check(e.L.tkv_pages_alloc(e.pages, 1, 2, ids.ctypes.data_as(u32p)))
    out = np.zeros(32 * 64, np.uint8)
    rc = e.L.tkv_pages_gather(e.pages, ids.ctypes.data_as(u32p), 2, 0, 32, out.ctypes.data_as(u8p), out.size)
    assert rc == 7  # unpopulated_page
    buf = np.full(32 * 64, 0xAB, np.uint8)
    check(e.L.tkv_pages_scatter(e.pages, buf.ctypes.data_as(u8p), buf.size, ids.ctypes.data_as(u32p), 2, 1, 32))
    rc = e.L.tkv_pages_gather(e.pages, ids.ctypes.data_as(u32p), 2, 0, 32, out.ctypes.data_as(u8p), out.size)
    assert rc == 7
    check(e.L.tkv_pages_gather(e.pages, ids.ctypes.data_as(u32p), 2, 1, 32, out.ctypes.data_as(u8p), out.size))
    small = np.zeros(3, np.uint8)
    assert e.L.tkv_pages_scatter(e.pages, small.ctypes.data_as(u8p), 3, ids.ctypes.data_as(u32p), 2, 0, 16) == 6
    big = np.zeros(64 * 64, np.uint8)
    assert e.L.tkv_pages_scatter(e.pages, big.ctypes.data_as(u8p), big.size, ids.ctypes.data_as(u32p), 2, 0, 64) == 6
    e.close()


def test_alloc_pages_atomic_and_conserving(tkv):
    """test_kv_core.cpp:98-133 — a failed allocation hands out nothing, the
    pool is conserved across alloc/release, concurrent holders get distinct
    page ids."""
    from paper_2510_09665_b200._lib import u32p
    e = _engine(tkv, 4, 64, 10)
    L = e.L
    assert L.tkv_pages_free_count(e.pages) == 10
    a = np.zeros(6, np.uint32)
    assert L.tkv_pages_alloc(e.pages, 1, 6, a.ctypes.data_as(u32p)) == 0
    assert L.tkv_pages_free_count(e.pages) == 4 and L.tkv_pages_allocated_count(e.pages) == 6
    big = np.zeros(5, np.uint32)
    assert L.tkv_pages_alloc(e.pages, 2, 5, big.ctypes.data_as(u32p)) == 3  # out_of_pages
    assert L.tkv_pages_free_count(e.pages) == 4  # nothing handed out on failure
    b = np.zeros(4, np.uint32)
    assert L.tkv_pages_alloc(e.pages, 2, 4, b.ctypes.data_as(u32p)) == 0
    assert L.tkv_pages_free_count(e.pages) == 0
    assert L.tkv_pages_release(e.pages, 1) == 6 and L.tkv_pages_free_count(e.pages) == 6
    L.tkv_pages_release(e.pages, 2)
    assert L.tkv_pages_free_count(e.pages) == 10 and L.tkv_pages_allocated_count(e.pages) == 0
    c, d = np.zeros(5, np.uint32), np.zeros(5, np.uint32)
    assert L.tkv_pages_alloc(e.pages, 3, 5, c.ctypes.data_as(u32p)) == 0
    assert L.tkv_pages_alloc(e.pages, 4, 5, d.ctypes.data_as(u32p)) == 0
    assert len(set(c.tolist()) | set(d.tolist())) == 10
    # admit (SimEngine::admit) is all-or-nothing too
    assert e.bind_pages(5, 16) == 3 and L.tkv_pages_free_count(e.pages) == 0
    e.close()


def test_layer_page_table_roundtrip(tkv):
    """test_kv_core.cpp:191-205 — bind_layer / layer_pages per (query, layer);
    unbound layers and unknown queries are empty; release clears them."""
    from paper_2510_09665_b200._lib import u32p
    e = _engine(tkv, 4, 64, 32)
    L = e.L
    ids = np.zeros(8, np.uint32)
    assert L.tkv_pages_alloc(e.pages, 5, 8, ids.ctypes.data_as(u32p)) == 0
    l0, l1 = ids[:4].copy(), ids[4:].copy()
    assert L.tkv_pages_bind_layer(e.pages, 5, 0, l0.ctypes.data_as(u32p), 4) == 0
    assert L.tkv_pages_bind_layer(e.pages, 5, 1, l1.ctypes.data_as(u32p), 4) == 0
    assert np.array_equal(e.layer_pages(5, 0), l0) and np.array_equal(e.layer_pages(5, 1), l1)
    assert e.layer_pages(5, 3).size == 0 and e.layer_pages(6, 0).size == 0
    L.tkv_pages_release(e.pages, 5)
    assert e.layer_pages(5, 0).size == 0
    e.close()


def _multi_layer_case(tkv, C, bpt, L, spans, seed, ppt=0, per_layer=False):
    """K1 then K2 over random page tables for several chunk descriptors and
    all layers in ONE launch each (per_layer: one launch per layer, the
    layerwise connector's shape), checked against the oracle's per-page
    memcpy restatement (paged_store.cpp:123-175)."""
    from paper_2510_09665_b200.api import XferDescC, plan_tiles
    from paper_2510_09665_b200._lib import check, lib
    rng = np.random.default_rng(seed)
    pt = 16
    page_bytes = pt * bpt
    n_pages = sum(L * ((s[1] - s[0] + pt - 1) // pt) for s in spans) + 8
    pool_h = rng.integers(0, 256, size=n_pages * page_bytes, dtype=np.uint8)
    perm = rng.permutation(n_pages).astype(np.int32)
    pool = torch.from_numpy(pool_h).cuda()
    descs, tables, chunks, used = [], [], [], 0
    for (start, end, rec) in spans:
        npg = (end - start + pt - 1) // pt
        first = start // pt
        tab = np.full((L, first + npg), -1, np.int32)
        for layer in range(L):
            tab[layer, first:] = perm[used:used + npg]
            used += npg
        tables.append(torch.from_numpy(tab).cuda())
        chunks.append(torch.zeros(L * rec * bpt, dtype=torch.uint8, device="cuda"))
    for (start, end, rec), tab, ch in zip(spans, tables, chunks):
        d = XferDescC()
        d.chunk = ch.data_ptr()
        d.layer_stride = rec * bpt
        d.table_dev = tab.data_ptr()
        d.table_stride = tab.shape[1]
        d.first_page = start // pt
        d.n_tokens = end - start
        descs.append(d)
    tb, ppt_used = plan_tiles(descs, pt, page_bytes, 1 if per_layer else L, ppt)
    arr = (XferDescC * len(descs))(*descs)
    d_descs = torch.frombuffer(bytearray(bytes(arr)), dtype=torch.uint8).cuda()
    d_tb = torch.from_numpy(tb.view(np.int32)).cuda()
    layout = tkv.api.PagedLayoutC(base=pool.data_ptr(), layer_base_dev=None, page_stride=page_bytes,
                                  plane_stride=0, token_stride=bpt, plane_bytes=bpt, n_planes=1,
                                  page_tokens=pt, bpt=bpt, shared_table=0)
    addr_or = 0
    for d in descs:
        addr_or |= d.chunk | d.layer_stride
    def launch(fn):
        for l0, nl in ([(layer, 1) for layer in range(L)] if per_layer else [(0, L)]):
            check(fn(ct.byref(layout), d_descs.data_ptr(), d_tb.data_ptr(), len(descs), int(tb[-1]), l0, nl,
                     ppt_used, addr_or, 0, None))

    launch(lib().tkv_gather_layers)
    torch.cuda.synchronize()
    for (start, end, rec), tab, ch in zip(spans, tables, chunks):
        got = ch.cpu().numpy()
        t = tab.cpu().numpy()
        for layer in range(L):
            want = C.gather_tokens(pool_h, page_bytes, t[layer, start // pt:], bpt, end - start)
            seg = got[layer * rec * bpt: layer * rec * bpt + (end - start) * bpt]
            assert np.array_equal(seg, want), (bpt, layer, start, end)
    # K2: scatter fresh chunk bytes back, compare the whole pool with the oracle.
    ref_pool = pool_h.copy()
    for (start, end, rec), tab, ch in zip(spans, tables, chunks):
        src = rng.integers(0, 256, size=L * rec * bpt, dtype=np.uint8)
        ch.copy_(torch.from_numpy(src))
        t = tab.cpu().numpy()
        for layer in range(L):
            C.scatter_tokens(ref_pool, page_bytes, t[layer, start // pt:], bpt, end - start,
                             src[layer * rec * bpt: layer * rec * bpt + (end - start) * bpt])
    launch(lib().tkv_scatter_layers)
    torch.cuda.synchronize()
    assert np.array_equal(pool.cpu().numpy(), ref_pool)


@pytest.mark.parametrize("bpt", [8, 12, 64, 512, 4096])
def test_multilayer_gather_scatter(tkv, C, bpt):
    spans = [(0, 256, 256), (256, 512, 256), (512, 600, 88), (768, 1000, 256)]  # last clips a record
    _multi_layer_case(tkv, C, bpt, 5, spans, seed=bpt)


@pytest.mark.parametrize("per_layer", [False, True])
@pytest.mark.parametrize("bpt", [16, 48, 64, 512, 4096])
def test_unit_kernel_gather_scatter(tkv, C, bpt, per_layer):
    """One page per tile with 16-byte rows: the unit kernel (<= 4 KiB page
    pieces, one warp each), launched over all layers and per layer; ragged
    spans, a clipped record, an empty descriptor between others."""
    spans = [(0, 256, 256), (256, 256, 256), (256, 512, 256), (512, 600, 88), (768, 1000, 256), (1024, 1031, 7)]
    _multi_layer_case(tkv, C, bpt, 5, spans, seed=100 + bpt, ppt=1, per_layer=per_layer)


def test_multilayer_small_tiles(tkv, C):
    _multi_layer_case(tkv, C, 512, 3, [(0, 256, 256), (256, 300, 256)], seed=5, ppt=3)


def test_vllm_two_plane_layout(tkv):
    """K/V planes per layer with a shared block table (vLLM layout): chunk row
    = K(h*D) | V(h*D). Checked against a numpy restatement."""
    from paper_2510_09665_b200.api import XferDescC, plan_tiles
    from paper_2510_09665_b200._lib import check, lib
    rng = np.random.default_rng(9)
    L, blocks, pt, hd = 3, 20, 16, 256  # plane bytes per token
    layers = [torch.from_numpy(rng.integers(0, 256, size=2 * blocks * pt * hd, dtype=np.uint8)).cuda()
              for _ in range(L)]
    bases = torch.tensor([t.data_ptr() for t in layers], dtype=torch.int64).cuda()
    table = rng.permutation(blocks).astype(np.int32)
    tab = torch.from_numpy(table).cuda()
    n_tok = 70
    ch = torch.zeros(L * n_tok * 2 * hd, dtype=torch.uint8, device="cuda")
    d = XferDescC(chunk=ch.data_ptr(), layer_stride=n_tok * 2 * hd, table_dev=tab.data_ptr(),
                  table_stride=blocks, first_page=0, n_tokens=n_tok)
    tb, ppt = plan_tiles([d], pt, pt * hd, L)
    d_descs = torch.frombuffer(bytearray(bytes(d)), dtype=torch.uint8).cuda()
    d_tb = torch.from_numpy(tb.view(np.int32)).cuda()
    layout = tkv.api.PagedLayoutC(base=0, layer_base_dev=bases.data_ptr(), page_stride=pt * hd,
                                  plane_stride=blocks * pt * hd, token_stride=hd, plane_bytes=hd, n_planes=2,
                                  page_tokens=pt, bpt=2 * hd, shared_table=1)
    check(lib().tkv_gather_layers(ct.byref(layout), d_descs.data_ptr(), d_tb.data_ptr(), 1, int(tb[-1]), 0, L,
                                  ppt, d.chunk | d.layer_stride, 0, None))
    torch.cuda.synchronize()
    got = ch.cpu().numpy().reshape(L, n_tok, 2, hd)
    for layer in range(L):
        kv = layers[layer].cpu().numpy().reshape(2, blocks, pt, hd)
        for t in range(n_tok):
            b = table[t // pt]
            assert np.array_equal(got[layer, t, 0], kv[0, b, t % pt])
            assert np.array_equal(got[layer, t, 1], kv[1, b, t % pt])


@pytest.mark.parametrize("nbytes,src_off,dst_off", [(0, 0, 0), (1, 0, 0), (4096 * 4 + 12, 0, 0),
                                                    (1000, 3, 0), (777, 16, 48), (1 << 20, 0, 16)])
def test_sm_copy_pinned_to_device(tkv, nbytes, src_off, dst_off):
    """tkv_sm_copy: exact bytes from pinned host memory into HBM (vector body +
    byte tail, or byte path when misaligned); nothing past the end is touched."""
    from paper_2510_09665_b200._lib import check, lib
    rng = np.random.default_rng(nbytes)
    host = torch.empty(nbytes + 64, dtype=torch.uint8, pin_memory=True)
    host.numpy()[:] = rng.integers(0, 256, size=nbytes + 64, dtype=np.uint8)
    dev = torch.full((nbytes + 128,), 0xAB, dtype=torch.uint8, device="cuda")
    check(lib().tkv_sm_copy(host.data_ptr() + src_off, dev.data_ptr() + dst_off, nbytes, None))
    torch.cuda.synchronize()
    d = dev.cpu().numpy()
    assert np.array_equal(d[dst_off:dst_off + nbytes], host.numpy()[src_off:src_off + nbytes])
    assert (d[:dst_off] == 0xAB).all() and (d[dst_off + nbytes:] == 0xAB).all()


@pytest.mark.parametrize("tp", [2, 4])
def test_tp_shards_are_head_slices(tkv, C, tp):
    """TP head sharding (a18): rank r's pool holds bytes [r*S, (r+1)*S) of
    every full KV row, S = bpt/tp. Each rank's compute + store + retrieve
    through its own connector; concatenating the ranks' retrieved rows gives
    the full-model rows of the oracle (synth_token_kv at bpt)."""
    from paper_2510_09665_b200.api import Engine
    full, L, n = 512, 3, 300
    S = full // tp
    prompt = rand_tokens(np.random.default_rng(40 + tp), n)
    rows = []
    for r in range(tp):
        e = Engine(num_layers=L, bpt=S, page_tokens=16, tag="tp-test", chunk_size=64, ram_slots=16,
                   num_pages=256, shard_offset=r * S)
        e.get_num_new_matched_tokens(1, prompt)
        e.bind_pages(1, n)
        e.update_state_after_alloc(1, (n + 15) // 16, 0)
        m = e.build_connector_meta([(1, prompt)])
        assert e.start_load_kv(m) == 0
        for layer in range(L):
            e.wait_load_kv(m, layer)
            e.compute_range(1, prompt, 0, n, layers=(layer, layer + 1))
            if layer:
                e.wait_store_kv(m, layer - 1)
            e.start_store_kv(m)
        assert e.wait_store_kv(m, L - 1) == 0
        e.finish_query(1)
        e.release_query(1)
        assert e.get_num_new_matched_tokens(2, prompt) == n - 1  # keys are rank-independent
        e.bind_pages(2, n)
        e.update_state_after_alloc(2, (n + 15) // 16, (n - 1 + 15) // 16)
        m = e.build_connector_meta([(2, prompt)])
        assert e.start_load_kv(m) == 0
        for layer in range(L):
            e.wait_load_kv(m, layer)
        e.synchronize()
        assert e.verify_range(2, prompt, 0, n - 1) == 0
        rows.append([e.gather_layer(2, layer, n - 1).reshape(n - 1, S) for layer in range(L)])
        e.close()
    seed = C.model_seed("tp-test")
    for layer in range(L):
        want = C.synth_layer_kv(seed, prompt[:n - 1], layer, 0, full).reshape(n - 1, full)
        got = np.concatenate([rows[r][layer] for r in range(tp)], axis=1)
        assert np.array_equal(got, want), layer


@pytest.mark.parametrize("direction", ["gather", "scatter"])
def test_vllm_slot_mapping(tkv, direction):
    """Per-token slot_mapping (vLLM: slot = block * block_size + offset, or any
    token -> slot map) is the paged layout with page_tokens = 1: the table is
    the slot mapping and a "page" is one token row. K/V planes per layer,
    scattered slots; gather (store) and scatter (retrieve) against numpy."""
    from paper_2510_09665_b200.api import XferDescC, plan_tiles
    from paper_2510_09665_b200._lib import check, lib
    rng = np.random.default_rng(13)
    L, n_slots, hd, n_tok = 3, 400, 128, 300  # hd = plane bytes per token (H*D*elt)
    kv = [torch.from_numpy(rng.integers(0, 256, size=2 * n_slots * hd, dtype=np.uint8)).cuda() for _ in range(L)]
    bases = torch.tensor([t.data_ptr() for t in kv], dtype=torch.int64).cuda()
    slots = rng.permutation(n_slots)[:n_tok].astype(np.int32)  # arbitrary, non-contiguous
    tab = torch.from_numpy(slots).cuda()
    ch = torch.from_numpy(rng.integers(0, 256, size=L * n_tok * 2 * hd, dtype=np.uint8)).cuda()
    d = XferDescC(chunk=ch.data_ptr(), layer_stride=n_tok * 2 * hd, table_dev=tab.data_ptr(),
                  table_stride=n_tok, first_page=0, n_tokens=n_tok)
    tb, ppt = plan_tiles([d], 1, hd, L)
    d_descs = torch.frombuffer(bytearray(bytes(d)), dtype=torch.uint8).cuda()
    d_tb = torch.from_numpy(tb.view(np.int32)).cuda()
    layout = tkv.api.PagedLayoutC(base=0, layer_base_dev=bases.data_ptr(), page_stride=hd,
                                  plane_stride=n_slots * hd, token_stride=hd, plane_bytes=hd, n_planes=2,
                                  page_tokens=1, bpt=2 * hd, shared_table=1)
    before = [t.cpu().numpy().reshape(2, n_slots, hd).copy() for t in kv]
    chunk_before = ch.cpu().numpy().reshape(L, n_tok, 2, hd).copy()
    fn = lib().tkv_gather_layers if direction == "gather" else lib().tkv_scatter_layers
    check(fn(ct.byref(layout), d_descs.data_ptr(), d_tb.data_ptr(), 1, int(tb[-1]), 0, L, ppt,
             d.chunk | d.layer_stride, 0, None))
    torch.cuda.synchronize()
    for layer in range(L):
        if direction == "gather":
            got = ch.cpu().numpy().reshape(L, n_tok, 2, hd)[layer]
            assert np.array_equal(got, before[layer][:, slots].transpose(1, 0, 2))
        else:
            want = before[layer].copy()
            want[:, slots] = chunk_before[layer].transpose(1, 0, 2)
            assert np.array_equal(kv[layer].cpu().numpy().reshape(2, n_slots, hd), want)


def test_bulk_variant_gather_scatter_subprocess():
    """The bulk-copy (cp.async.bulk) variant of the unit kernel is selected
    by an environment switch read once per process: run the unit-kernel
    parity cases in a child process with TKV_PAGED_KERNEL=bulk."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, TKV_PAGED_KERNEL="bulk")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu",
                        "tests/test_gpu_kernels.py::test_unit_kernel_gather_scatter",
                        "tests/test_gpu_kernels.py::test_vllm_slot_mapping"],
                       cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


def test_unit_kernel_many_descriptors(tkv, C):
    """More descriptors than the unit kernel keeps in shared memory (4096):
    the descriptor search runs on the global prefix. 4500 one-page
    descriptors (ragged: 1-16 tokens), one-layer launches per layer."""
    rng = np.random.default_rng(4500)
    spans = [(0, int(rng.integers(1, 17)), 16) for _ in range(4500)]  # each its own one-page table
    _multi_layer_case(tkv, C, 64, 2, spans, seed=4501, ppt=1, per_layer=True)


def _affine_descs(n_chunks, last_tokens, pt, bpt, L, chunk0, table_dev, table_stride, first_page, rec=256):
    from paper_2510_09665_b200.api import XferDescC
    out = []
    for i in range(n_chunks):
        d = XferDescC()
        d.chunk = chunk0 + i * L * rec * bpt
        d.layer_stride = rec * bpt
        d.table_dev = table_dev
        d.table_stride = table_stride
        d.first_page = first_page + i * (rec // pt)
        d.n_tokens = rec if i + 1 < n_chunks else last_tokens
        out.append(d)
    return out


@pytest.mark.parametrize("bpt,last,shared,layer_base", [(4096, 256, False, False), (512, 88, False, False),
                                                         (16, 7, True, False), (1024, 200, False, True),
                                                         (48, 256, True, True)])
def test_affine_launches_match_oracle(tkv, C, bpt, last, shared, layer_base):
    """The affine launch form (one query's consecutive chunks): K1 per layer
    and over all layers, K2 back, against the oracle's per-page memcpy
    restatement — full and ragged last chunk, a shared (layer-independent)
    page table, per-layer pool bases."""
    from paper_2510_09665_b200._lib import AffinePlanC, XferDescC, check, lib
    rng = np.random.default_rng(bpt + last)
    pt, L, n_chunks, first = 16, 3, 4, 2
    page_bytes = pt * bpt
    pages_q = first + (n_chunks * 256) // pt
    n_pages = L * pages_q + 8
    pool_h = rng.integers(0, 256, size=n_pages * page_bytes, dtype=np.uint8)
    perm = rng.permutation(n_pages).astype(np.int32)
    rows = 1 if shared else L
    tab = perm[:rows * pages_q].reshape(rows, pages_q).copy()
    if layer_base:  # per-layer pools: layer l's page p at bases[l] + p * page_bytes (one pool, offset bases)
        pool = torch.from_numpy(np.concatenate([pool_h] * L)).cuda()
        bases = torch.tensor([pool.data_ptr() + l * n_pages * page_bytes for l in range(L)], dtype=torch.int64).cuda()
        host_pool = [pool_h] * L
    else:
        pool = torch.from_numpy(pool_h).cuda()
        bases = None
        host_pool = [pool_h] * L
    d_tab = torch.from_numpy(tab).cuda()
    ch = torch.zeros(n_chunks * L * 256 * bpt, dtype=torch.uint8, device="cuda")
    descs = _affine_descs(n_chunks, last, pt, bpt, L, ch.data_ptr(), d_tab.data_ptr(), pages_q, first)
    arr = (XferDescC * n_chunks)(*descs)
    plan = AffinePlanC()
    assert lib().tkv_affine_form(ct.cast(arr, ct.c_void_p), n_chunks, pt, ct.byref(plan)) == 0
    assert plan.pages_per_desc == 16 and plan.last_tokens == last and plan.chunk_stride == L * 256 * bpt
    layout = tkv.api.PagedLayoutC(base=0 if layer_base else pool.data_ptr(),
                                  layer_base_dev=bases.data_ptr() if layer_base else None, page_stride=page_bytes,
                                  plane_stride=0, token_stride=bpt, plane_bytes=bpt, n_planes=1, page_tokens=pt,
                                  bpt=bpt, shared_table=int(shared))

    def want_chunks(pools):
        out = np.zeros(ch.numel(), np.uint8)
        for i in range(n_chunks):
            n = 256 if i + 1 < n_chunks else last
            for layer in range(L):
                t = tab[0 if shared else layer, first + i * 16:]
                o = i * L * 256 * bpt + layer * 256 * bpt
                out[o:o + n * bpt] = C.gather_tokens(pools[layer], page_bytes, t, bpt, n)
        return out
    for per_layer in (True, False):
        ch.zero_()
        for l0, nl in ([(layer, 1) for layer in range(L)] if per_layer else [(0, L)]):
            check(lib().tkv_gather_layers_affine(ct.byref(layout), ct.byref(plan), l0, nl, 0, None))
        torch.cuda.synchronize()
        assert np.array_equal(ch.cpu().numpy(), want_chunks(host_pool)), per_layer
    # K2: fresh chunk bytes back into the pages
    src = rng.integers(0, 256, size=ch.numel(), dtype=np.uint8)
    ch.copy_(torch.from_numpy(src))
    ref = [p.copy() for p in ([pool_h] if not layer_base else [pool_h.copy() for _ in range(L)])]
    for i in range(n_chunks):
        n = 256 if i + 1 < n_chunks else last
        for layer in range(L):
            t = tab[0 if shared else layer, first + i * 16:]
            o = i * L * 256 * bpt + layer * 256 * bpt
            C.scatter_tokens(ref[layer if layer_base else 0], page_bytes, t, bpt, n, src[o:o + n * bpt])
    for layer in range(L):
        check(lib().tkv_scatter_layers_affine(ct.byref(layout), ct.byref(plan), layer, 1, 0, None))
    torch.cuda.synchronize()
    got = pool.cpu().numpy()
    if layer_base:
        for layer in range(L):
            assert np.array_equal(got[layer * n_pages * page_bytes:(layer + 1) * n_pages * page_bytes], ref[layer])
    else:
        assert np.array_equal(got, ref[0])
