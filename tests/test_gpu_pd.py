"""PD disaggregation on the B200 (run_pd, src/sim_engine.cpp:347-543): the
prefiller's pages are gathered chunk by chunk straight into the decoder's
landing buffer (K1 writing device memory — a peer GPU's in production, the
same GPU here since gpurun gives one), ordinals are pushed out of order with
a duplicate, the decoder awaits them in order and scatters all chunks into
its own pages with one K2 launch. Byte oracle: the reference's own PD check,
synth_layer_kv recomputation of every layer (sim_engine.cpp:474-490)."""
import numpy as np
import pytest
import torch

import scenarios as S

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("late", [False, True])
@pytest.mark.parametrize("staged", [False, True])
def test_pd_send_land_byte_exact(tkv, C, staged, late):
    """staged: K1 into local staging + copy-engine peer copies in groups (the
    group size is forced down so the 7 chunks travel as several copies).
    late: the engine stream runs ~1 ms behind the host before the compute,
    so the send, the await and the land must all be ordered by the streams,
    not by luck."""
    from paper_2510_09665_b200.api import Engine, PdStaging, pd_land, pd_send, pd_send_staged
    spec = dict(num_layers=4, bpt=512, page_tokens=16, tag="pd-test", chunk_size=32)
    pre = Engine(**spec, ram_slots=4, num_pages=256)
    dec = Engine(**spec, ram_slots=4, num_pages=256)
    prompt = S.make_prompt(200, 71)  # 7 chunks, the last one partial (8 tokens)
    pre.bind_pages(10, 200)
    if late:
        torch.cuda._sleep(2_000_000)
    pre.compute_range(10, prompt, 0, 200)
    stride = 4 * 32 * 512
    landing = torch.zeros(7 * stride, dtype=torch.uint8, device="cuda")
    staging = PdStaging()
    assert staging.register_query(10) == 0
    if staged:
        buf = torch.zeros(7 * stride, dtype=torch.uint8, device="cuda")
        recs = pd_send_staged(pre, 10, 200, landing.data_ptr(), stride, buf.data_ptr(), group_bytes=2 * stride)
    else:
        recs = pd_send(pre, 10, 200, landing.data_ptr(), stride)
    assert [r.token_count for r in recs] == [32] * 6 + [8]
    for o in [3, 0, 6, 1, 5, 2, 4, 3]:
        assert staging.push(10, o, o == 6, recs[o]) == 0
    rc, landed = staging.await_(10)
    assert rc == 0 and [r.first_token for r in landed] == [32 * i for i in range(7)]
    dec.bind_pages(10, 200)
    pd_land(dec, 10, landed)
    assert S.pages_equal_synth(dec, 10, prompt, 200, C)
    # the landed chunk payloads are the KVChunk byte contract [L][T][bpt]
    seed = C.model_seed("pd-test")
    host = landing.cpu().numpy()
    for i, r in enumerate(recs):
        want = C.synth_chunk(seed, prompt, 32 * i, r.token_count, 4, 512)
        assert np.array_equal(host[i * stride: i * stride + want.size], want)
    pre.close()
    dec.close()


def test_pd_land_rejects_bad_records(tkv):
    from paper_2510_09665_b200.api import Engine, PdRecordC, pd_land
    from paper_2510_09665_b200._lib import TkvError
    dec = Engine(num_layers=2, bpt=64, page_tokens=16, tag="pd-test", chunk_size=32, ram_slots=2,
                 num_pages=64)
    dec.bind_pages(1, 64)
    buf = torch.zeros(4096, dtype=torch.uint8, device="cuda")
    with pytest.raises(TkvError) as e:  # size does not match the geometry (sim_engine.cpp:461-462)
        pd_land(dec, 1, [PdRecordC(addr=buf.data_ptr(), bytes=100, token_count=32, first_token=0)])
    assert e.value.code == 6
    with pytest.raises(TkvError) as e:  # beyond the query's pages
        pd_land(dec, 1, [PdRecordC(addr=buf.data_ptr(), bytes=2 * 32 * 64, token_count=32, first_token=64)])
    assert e.value.code == 6
    dec.close()


def _ipc_child(handle: bytes, offset: int, n: int, q):
    """Second process: map the exported buffer and write a pattern into it."""
    import ctypes as ct
    import torch
    from paper_2510_09665_b200._lib import lib
    torch.cuda.set_device(0)
    h = (ct.c_uint8 * 64).from_buffer_copy(handle)
    ptr = ct.c_void_p()
    rc = lib().tkv_ipc_open_handle(h, offset, ct.byref(ptr))
    if rc == 0:
        src = torch.arange(n, dtype=torch.int64, device="cuda").to(torch.uint8) ^ 0x5A
        rc = lib().tkv_ce_copy(ct.c_void_p(src.data_ptr()), ptr, n, None)
        torch.cuda.synchronize()
        lib().tkv_ipc_close(ptr, offset)
    q.put(rc)


def test_pd_ipc_handle_suballocation(tkv):
    """The cross-process landing path with a buffer carved out of a larger
    allocation (what a caching allocator hands out): the handle maps the
    allocation base, the offset travels beside it, and the other process's
    writes land exactly in the sub-buffer."""
    import ctypes as ct
    import multiprocessing as mp
    from paper_2510_09665_b200._lib import lib
    big = torch.zeros(4 << 20, dtype=torch.uint8, device="cuda")
    off0, n = 3 * 4096 + 256, 1 << 20
    buf = big[off0:off0 + n]
    h = (ct.c_uint8 * 64)()
    offset = ct.c_uint64(0)
    assert lib().tkv_ipc_get_handle(ct.c_void_p(buf.data_ptr()), h, ct.byref(offset)) == 0
    assert offset.value >= off0  # at least the carve-out; more if torch's segment is shared
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_ipc_child, args=(bytes(h), offset.value, n, q))
    p.start()
    rc = q.get(timeout=120)
    p.join(timeout=60)
    assert rc == 0
    want = (torch.arange(n, dtype=torch.int64, device="cuda").to(torch.uint8) ^ 0x5A)
    assert torch.equal(buf, want)
    assert int(big[:off0].count_nonzero()) == 0 and int(big[off0 + n:].count_nonzero()) == 0


@pytest.mark.parametrize("late", [False, True])
def test_pd_layer_streamed_page_and_chunk_granularity(tkv, C, late):
    """run_pd at page granularity (one record per 16-token window,
    src/sim_engine.cpp:398-424, landed per window :457-472) and at chunk
    granularity, both sent layer by layer while the prefill computes (each
    layer's K1 ordered after the engine stream's compute of it): the decoder
    pages equal the recomputation (the reference's PD byte oracle,
    sim_engine.cpp:474-490) and each other — the disaggregated run equals the
    monolithic one (tests/test_engine.cpp:412-456) — with ceil(len/16) and
    ceil(len/32) messages. late: the engine stream runs ~1 ms behind the host
    before every layer, so only the events order the sends."""
    from paper_2510_09665_b200.api import Engine, PdLayerSender, PdStaging, pd_land
    L, bpt, pt, cs, n = 4, 512, 16, 32, 200
    spec = dict(num_layers=L, bpt=bpt, page_tokens=pt, tag="pd-test", chunk_size=cs)
    stream = torch.cuda.Stream()
    pre = Engine(**spec, ram_slots=4, num_pages=256, stream=stream)
    prompt = S.make_prompt(n, 73)
    pre.bind_pages(20, n)
    images = {}
    for unit in (pt, cs):
        stride = L * unit * bpt
        n_units = (n + unit - 1) // unit
        landing = torch.zeros(n_units * stride, dtype=torch.uint8, device="cuda")
        torch.cuda.synchronize()  # the sender's own stream is not ordered after torch's fill
        snd = PdLayerSender(pre, 20, n, unit, landing.data_ptr(), stride)
        for layer in range(L):
            if late:
                with torch.cuda.stream(stream):
                    torch.cuda._sleep(2_000_000)
            pre.compute_range(20, prompt, 0, n, layers=(layer, layer + 1))
            assert snd.layer(layer) == 0
        assert snd.layer(0) == 4  # duplicate_key: a layer goes once
        recs = snd.finish()
        snd.close()
        assert len(recs) == n_units  # messages: 13 windows, 7 chunks
        assert [r.first_token for r in recs] == [unit * i for i in range(n_units)]
        assert [r.token_count for r in recs] == [min(unit, n - unit * i) for i in range(n_units)]
        staging = PdStaging()
        assert staging.register_query(20) == 0
        order = list(range(n_units))[::-1] + [n_units // 2]  # out of order + a duplicate
        for o in order:
            assert staging.push(20, o, o == n_units - 1, recs[o]) == 0
        rc, landed = staging.await_(20)
        assert rc == 0 and len(landed) == n_units
        dec = Engine(**spec, ram_slots=4, num_pages=256)
        dec.bind_pages(20, n)
        pd_land(dec, 20, landed)
        assert S.pages_equal_synth(dec, 20, prompt, n, C)
        images[unit] = S.page_image(dec, 20, n)
        # a window record is the layer-major slice of its window [L][T][bpt]
        host = landing.cpu().numpy()
        seed = C.model_seed("pd-test")
        for i in (0, n_units - 1):
            want = C.synth_chunk(seed, prompt, unit * i, recs[i].token_count, L, bpt)
            assert np.array_equal(host[i * stride: i * stride + want.size], want)
        dec.close()
    assert images[pt] == images[cs]
    # sending a layer the engine has not computed is refused (check_readable)
    pre.bind_pages(21, n)
    buf = torch.zeros(L * n * bpt, dtype=torch.uint8, device="cuda")
    torch.cuda.synchronize()
    snd = PdLayerSender(pre, 21, n, pt, buf.data_ptr(), L * pt * bpt)
    assert snd.layer(0) == 7  # unpopulated_page
    assert snd.layer(L) == 16  # invalid_argument: out of range
    snd.close()
    pre.close()


def test_c5_loopback_config_small():
    """bench.py's configs.c5_loopback at a small size: every send path, the
    PdStaging contract and the land run and the landed page image is exact."""
    import os
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
    import bench_configs
    r = bench_configs.c5_loopback(reps=1, cpu=False, n=1000, L=4)
    assert r["verify"]["page_mismatch_words"] == 0 and r["verify"]["chunks_landed"] == 4, r
    assert r["sm_direct_gbps"] > 0 and r["ce_staged_gbps"] > 0 and r["layer_streamed_page_gbps"] > 0
