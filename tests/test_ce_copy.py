"""Host-tier copy-engine pieces (csrc/ce_copy.cpp): the grouping of a layer's
chunk slices into pitched runs (CPU, no device call), and on the GPU the
copies themselves, byte-exact for ascending / descending / broken runs, mixed
widths and empty pieces, both directions."""
import ctypes as ct

import numpy as np
import pytest

PMAX = 1 << 31


def _plan(L, dst, src, sizes, pmax=PMAX):
    n = len(sizes)
    D = (ct.c_void_p * max(n, 1))(*dst)
    S = (ct.c_void_p * max(n, 1))(*src)
    Z = (ct.c_size_t * max(n, 1))(*sizes)
    first = (ct.c_size_t * max(n, 1))()
    rows = (ct.c_size_t * max(n, 1))()
    k = L.tkv_plan_copy_runs(D, S, Z, n, pmax, first, rows)
    return [(int(first[i]), int(rows[i])) for i in range(k)]


def _model(dst, src, sizes, pmax=PMAX):
    """The grouping rule restated: greedy runs of one width whose two
    addresses move by the run's first step (same sign, >= width, <= pmax)."""
    runs, i, n = [], 0, len(sizes)
    while i < n:
        w, j = sizes[i], i + 1
        sp = dp = 0
        if w > 0 and j < n and sizes[j] == w:
            sp, dp = src[j] - src[i], dst[j] - dst[i]
            ok = (sp >= w and dp >= w) or (sp <= -w and dp <= -w)
            if ok and abs(sp) <= pmax and abs(dp) <= pmax:
                j += 1
                while j < n and sizes[j] == w and src[j] - src[j - 1] == sp and dst[j] - dst[j - 1] == dp:
                    j += 1
        runs.append((i if j - i == 1 or sp > 0 else j - 1, j - i))
        i = j
    return runs


def test_runs_of_consecutive_slots(tkv):
    L = tkv.lib()
    slot, w, ring = 80 << 20, 1 << 20, 1 << 40
    base = 1 << 36
    # 64 consecutive slots into a packed ring: one run
    src = [base + i * slot for i in range(64)]
    dst = [ring + i * w for i in range(64)]
    assert _plan(L, dst, src, [w] * 64) == [(0, 64)]
    # descending slots into a descending ring order: one run read from the last piece
    assert _plan(L, dst[::-1], src[::-1], [w] * 64) == [(63, 64)]
    # descending slots into an ascending ring: no run (mixed signs)
    assert _plan(L, dst, src[::-1], [w] * 64) == [(i, 1) for i in range(64)]
    # a gap in the slots splits the run
    src2 = src[:10] + [s + slot for s in src[10:]]
    assert _plan(L, dst, src2, [w] * 64) == [(0, 10), (10, 54)]
    # a short last piece (ragged tail chunk) stands alone
    assert _plan(L, dst, src, [w] * 63 + [w // 2]) == [(0, 63), (63, 1)]
    # overlapping rows (step below the width) never form a run
    assert _plan(L, [ring + i * (w // 2) for i in range(4)], src[:4], [w] * 4) == [(i, 1) for i in range(4)]
    # pitch above the limit: every piece alone
    assert _plan(L, dst[:8], src[:8], [w] * 8, pmax=slot - 1) == [(i, 1) for i in range(8)]
    assert _plan(L, [], [], []) == []


def test_runs_match_model_random(tkv):
    L = tkv.lib()
    rng = np.random.default_rng(7)
    for trial in range(300):
        n = int(rng.integers(1, 40))
        w = int(rng.choice([0, 16, 4096, 1 << 20]))
        slot = w * int(rng.integers(1, 5)) + int(rng.choice([0, 0, 16]))
        order = rng.permutation(n) if trial % 3 == 0 else (np.arange(n)[::-1] if trial % 3 == 1 else np.arange(n))
        if trial % 5 == 0:  # runs broken at random places
            order = np.concatenate([np.sort(c) for c in np.array_split(order, int(rng.integers(1, 5)))])
        src = [(1 << 36) + int(o) * max(slot, 1) for o in order]
        sizes = [w if rng.random() > 0.1 else w // 2 for _ in range(n)]
        dst, off = [], 1 << 40
        for i in range(n):
            dst.append(off)
            off += sizes[i]
        if trial % 7 == 0:
            dst = dst[::-1]
        pmax = int(rng.choice([PMAX, max(slot, 1), max(slot, 1) - 1]))
        assert _plan(L, dst, src, sizes, pmax) == _model(dst, src, sizes, pmax), trial


@pytest.mark.gpu
def test_ce_copy_pieces_byte_exact(tkv):
    import torch
    L = tkv.lib()
    slot, w, nslots = 40 << 10, 8 << 10, 48
    host = torch.empty(slot * nslots, dtype=torch.uint8, pin_memory=True)
    host.copy_(torch.randint(0, 256, (slot * nslots,), dtype=torch.uint8))
    rng = np.random.default_rng(3)
    s = torch.cuda.Stream()
    for case in ["ascending", "descending", "mixed", "random", "ragged", "slab_end", "slab_end_down"]:
        n = 32
        # slab_end*: the run ends on the allocation's last slot, first layer of
        # the slot, so pitch x rows reaches past the allocation
        slots = {"ascending": np.arange(n), "descending": np.arange(n)[::-1],
                 "slab_end": np.arange(nslots - n, nslots), "slab_end_down": np.arange(nslots - n, nslots)[::-1],
                 "mixed": np.concatenate([np.arange(10), np.arange(30, 20, -1), np.arange(36, 48)]),
                 "random": rng.permutation(nslots)[:n], "ragged": np.arange(n)}[case]
        n = len(slots)
        layer = 0 if case.startswith("slab_end") else int(rng.integers(0, slot // w))
        sizes = [w] * n if case != "ragged" else [int(x) for x in rng.choice([0, 16, w // 2, w], size=n)]
        offs = np.concatenate([[0], np.cumsum(sizes)[:-1]]).astype(np.int64)
        if case in ("descending", "slab_end_down"):  # ring order follows the (descending) slot order
            offs = offs[::-1].copy()
        ring = torch.zeros(int(sum(sizes)) + 64, dtype=torch.uint8, device="cuda")
        hsrc = [host.data_ptr() + int(sl) * slot + layer * w for sl in slots]
        ddst = [ring.data_ptr() + int(o) for o in offs]
        D = (ct.c_void_p * n)(*ddst)
        S = (ct.c_void_p * n)(*hsrc)
        Z = (ct.c_size_t * n)(*sizes)
        rc = L.tkv_ce_copy_pieces(D, S, Z, n, 1, ct.c_void_p(s.cuda_stream))
        assert rc == 0, (case, "h2d", L.tkv_last_error())
        s.synchronize()
        got = ring.cpu().numpy()
        hn = host.numpy()
        for i in range(n):
            a = int(slots[i]) * slot + layer * w
            assert np.array_equal(got[offs[i]:offs[i] + sizes[i]], hn[a:a + sizes[i]]), (case, i)
        # and back: D2H into a fresh host image at the same slots
        back = torch.zeros(host.shape, dtype=torch.uint8, pin_memory=True)
        D = (ct.c_void_p * n)(*[back.data_ptr() + int(sl) * slot + layer * w for sl in slots])
        S = (ct.c_void_p * n)(*ddst)
        rc = L.tkv_ce_copy_pieces(D, S, Z, n, 2, ct.c_void_p(s.cuda_stream))
        assert rc == 0, (case, "d2h", L.tkv_last_error())
        s.synchronize()
        bn = back.numpy()
        for i in range(n):
            a = int(slots[i]) * slot + layer * w
            assert np.array_equal(bn[a:a + sizes[i]], hn[a:a + sizes[i]]), (case, "d2h", i)
        written = sum(sizes)
        assert int(np.count_nonzero(bn)) <= written


@pytest.mark.gpu
def test_reverse_evictions_keep_pitched_runs(tkv, C):
    """A batch whose LRU victims free slots in descending order still writes
    (and later reads) its full chunks as one pitched run per layer: the store
    hands a batch's slots out in ascending order (store.cpp
    begin_write_batch). Bytes checked against synth after the reload."""
    import scenarios as S
    from paper_2510_09665_b200.api import Engine
    cs, L = S.CONN["chunk_size"], S.CONN["num_layers"]
    e = Engine(**S.CONN, ram_slots=8, num_pages=512)
    state = {"qid": 1}

    def serve(p):
        q = state["qid"]
        state["qid"] += 1
        m_ = e.get_num_new_matched_tokens(q, p)
        e.bind_pages(q, len(p))
        e.update_state_after_alloc(q, (len(p) + 15) // 16, (m_ + 15) // 16)
        m = e.build_connector_meta([(q, p)])
        S.transfer(e, m, q, p)
        ok = S.pages_equal_synth(e, q, p, len(p), C)
        e.drop_meta(m)
        e.finish_query(q)
        e.release_query(q)
        return m_, ok

    singles = [S.make_prompt(cs, 500 + i) for i in range(8)]
    for p in singles:  # slots 0..7
        assert serve(p) == (0, True)
    for p in singles[::-1]:  # touched 7 first: LRU victims come out 7, 6, 5, ...
        assert serve(p) == (cs - 1, True)
    q = S.make_prompt(4 * cs + 1, 900)  # 4 full chunks + a 1-token tail
    p0, c0 = e.copy_runs()
    assert serve(q) == (0, True)  # stores 5 chunks into slots 7..3
    p1, c1 = e.copy_runs()
    assert p1 - p0 == 5 * L
    assert c1 - c0 == 2 * L, (p1 - p0, c1 - c0)  # full chunks one run, the tail alone
    assert serve(q) == (4 * cs, True)  # loads the 4 full chunks
    p2, c2 = e.copy_runs()
    assert p2 - p1 == 4 * L and c2 - c1 == L, (p2 - p1, c2 - c1)
    e.close()
