"""CPU: the PD landing/ordering contract (PdStaging, src/pd_staging.cpp)
driven through the C-ABI, compared with the unmodified reference PdStaging
on the same push sequences, plus the two-process (gloo, world_size 2)
prefiller -> decoder control plane of the NVLink PD path."""
import os
import threading
import time

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _ref_pd():
    import oracle
    if not oracle.ref_available():
        return None
    return oracle.Ref().lib


def _run_sequence(push, register, await_, cancel, seq):
    out = []
    for op in seq:
        if op[0] == "reg":
            out.append(("reg", register(op[1])))
        elif op[0] == "push":
            _, q, o, last = op
            out.append(("push", push(q, o, last)))
        elif op[0] == "await":
            out.append(("await",) + tuple(await_(op[1])))
        elif op[0] == "cancel":
            out.append(("cancel", cancel(op[1])))
    return out


SEQS = {
    # test_netcache.cpp:241-283: out of order with a duplicate
    "out_of_order": [("reg", 42)] + [("push", 42, o, o == 5) for o in [3, 0, 5, 1, 4, 2, 3]] + [("await", 42)],
    # test_netcache.cpp:285-306: ordinal abuse
    "abuse": [("reg", 1), ("reg", 1), ("push", 1, 2, True), ("push", 1, 5, False), ("push", 1, 0, False),
              ("push", 1, 1, False), ("await", 1), ("await", 99)],
    "final_below_filled": [("reg", 3), ("push", 3, 4, False), ("push", 3, 2, True), ("push", 3, 5, True),
                           ("push", 3, 0, False)],
    "unknown": [("push", 777, 0, True), ("cancel", 777)],
}


def _ours():
    from paper_2510_09665_b200.api import PdRecordC, PdStaging
    s = PdStaging()

    def push(q, o, last):
        return s.push(q, o, last, PdRecordC(addr=1000 + o, bytes=o, token_count=o, first_token=0))

    def await_(q):
        rc, recs = s.await_(q)
        return rc, [r.addr - 1000 for r in recs]
    return s, push, s.register_query, await_, s.cancel


def _reference():
    import ctypes as ct
    lib = _ref_pd()
    h = lib.ref_pd_create()

    def push(q, o, last):
        rec = (ct.c_uint8 * 1)(o)
        return lib.ref_pd_push(h, q, o, int(last), rec, 1)

    def await_(q):
        tags = (ct.c_uint8 * 256)()
        n = ct.c_size_t(0)
        rc = lib.ref_pd_await(h, q, tags, 256, ct.byref(n))
        return rc, [tags[i] for i in range(n.value)] if rc == 0 else []
    return h, push, lambda q: lib.ref_pd_register(h, q), await_, lambda q: lib.ref_pd_cancel(h, q)


@pytest.mark.parametrize("name", list(SEQS))
def test_pd_staging_matches_reference(tkv, name):
    if _ref_pd() is None:
        pytest.skip("oracle/_ref not built")
    s, *ours = _ours()
    h, *ref = _reference()
    assert _run_sequence(*ours, SEQS[name]) == _run_sequence(*ref, SEQS[name])
    _ref_pd().ref_pd_destroy(h)


def test_pd_staging_literal_expectations(tkv):
    s, push, register, await_, cancel = _ours()
    r = _run_sequence(push, register, await_, cancel, SEQS["out_of_order"])
    assert all(x[1] == 0 for x in r[:-1])
    assert r[-1] == ("await", 0, [0, 1, 2, 3, 4, 5])
    assert s.registered() == 0
    r = _run_sequence(push, register, await_, cancel, SEQS["abuse"])
    assert [x[1] for x in r] == [0, 4, 0, 14, 0, 0, 0, 10]  # duplicate_key, protocol_error, unknown_query


def test_pd_cancel_wakes_awaiter(tkv):
    s, push, register, await_, cancel = _ours()
    assert register(2) == 0
    t = threading.Thread(target=lambda: (time.sleep(0.05), cancel(2)))
    t.start()
    rc, recs = await_(2)
    t.join()
    assert rc == 15 and recs == []  # io_error "query cancelled"


# ---------------------------------------------------------- two processes --

def _pd_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n_chunks = 9
        if rank == 0:  # prefiller: send ordinals out of order with duplicates
            order = [4, 0, 8, 2, 1, 7, 3, 6, 5, 2, 8]
            for o in order:
                msg = torch.tensor([77, o, int(o == n_chunks - 1), 4096 * o, 256], dtype=torch.int64)
                dist.send(msg, dst=1)
            dist.send(torch.tensor([-1, 0, 0, 0, 0], dtype=torch.int64), dst=1)
        else:  # decoder: land into PdStaging, then await in ordinal order
            from paper_2510_09665_b200.api import PdRecordC, PdStaging
            s = PdStaging()
            assert s.register_query(77) == 0
            codes = []
            while True:
                msg = torch.zeros(5, dtype=torch.int64)
                dist.recv(msg, src=0)
                if msg[0] < 0:
                    break
                rec = PdRecordC(addr=int(msg[3]), bytes=0, token_count=int(msg[4]), first_token=int(msg[1]) * 256)
                codes.append(s.push(int(msg[0]), int(msg[1]), bool(msg[2]), rec))
            rc, recs = s.await_(77)
            q.put((codes, rc, [r.first_token for r in recs], [r.addr for r in recs]))
    finally:
        dist.destroy_process_group()


def test_pd_two_process_gloo(tkv):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29000 + os.getpid() % 1000
    procs = [ctx.Process(target=_pd_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    codes, rc, firsts, addrs = q.get(timeout=120)
    for p in procs:
        p.join(60)
    assert all(c == 0 for c in codes)
    assert rc == 0
    assert firsts == [256 * i for i in range(9)]
    assert addrs == [4096 * i for i in range(9)]


def _random_pd_sequence(rng):
    """Registrations (sometimes twice), pushes of shuffled ordinals with
    duplicates, several or no final flags, ordinals past the final, pushes
    for unknown queries; every query is cancelled before it is awaited (an
    incomplete await blocks by contract), and some are re-registered after."""
    seq = []
    qs = [int(q) for q in rng.choice(50, size=int(rng.integers(1, 4)), replace=False)]
    for q in qs:
        seq.append(("reg", q))
        if rng.random() < 0.2:
            seq.append(("reg", q))
    for _ in range(int(rng.integers(0, 14))):
        q = qs[int(rng.integers(len(qs)))] if rng.random() < 0.9 else 100 + int(rng.integers(5))
        seq.append(("push", q, int(rng.integers(0, 8)), bool(rng.random() < 0.2)))
    for q in qs:
        seq.append(("cancel", q))
        seq.append(("await", q))
        if rng.random() < 0.3:
            seq += [("reg", q), ("push", q, 0, True), ("await", q)]
    return seq


def test_pd_staging_random_sequences_match_reference(tkv):
    """300 random push/cancel sequences through both PdStaging
    implementations, every return code and every awaited ordinal list equal."""
    import numpy as np
    if _ref_pd() is None:
        pytest.skip("oracle/_ref not built")
    rng = np.random.default_rng(2510)
    for i in range(300):
        seq = _random_pd_sequence(rng)
        s, *ours = _ours()
        h, *ref = _reference()
        assert _run_sequence(*ours, seq) == _run_sequence(*ref, seq), (i, seq)
        _ref_pd().ref_pd_destroy(h)
