"""CPU: the connector's parallel host copy (csrc/host_copy.cpp) — the prompt
copies of every lookup go through it. Byte-exact against numpy for sizes
around the parallel threshold and the piece size, unaligned ends, and
several threads copying at once (one of them gets the helpers, the others
copy alone)."""
import ctypes as ct
import threading

import numpy as np


def _copy(L, dst, src, n, doff=0, soff=0):
    L.tkv_host_copy(ct.c_void_p(dst.ctypes.data + doff), ct.c_void_p(src.ctypes.data + soff), n)


def test_host_copy_sizes_and_alignments(tkv):
    L = tkv.lib()
    rng = np.random.default_rng(1)
    for n in [0, 1, 15, 16, 4095, 128 << 10, (128 << 10) - 1, (128 << 10) + 1, 64 << 10, (64 << 10) * 7 + 3,
              512 << 10, (1 << 20) + 17, 3 << 20]:
        for doff, soff in [(0, 0), (1, 0), (0, 3), (7, 5)]:
            src = rng.integers(0, 256, size=n + 16, dtype=np.uint8)
            dst = np.zeros(n + 16, np.uint8)
            _copy(L, dst, src, n, doff, soff)
            assert np.array_equal(dst[doff:doff + n], src[soff:soff + n]), (n, doff, soff)
            assert not dst[:doff].any() and not dst[doff + n:].any()


def test_host_copy_concurrent_callers(tkv):
    L = tkv.lib()
    n = 700 << 10
    srcs = [np.random.default_rng(i).integers(0, 256, size=n, dtype=np.uint8) for i in range(6)]
    dsts = [np.zeros(n, np.uint8) for _ in range(6)]
    errs = []

    def work(i):
        try:
            for _ in range(20):
                dsts[i][:] = 0
                _copy(L, dsts[i], srcs[i], n)
                assert np.array_equal(dsts[i], srcs[i])
        except AssertionError as e:  # pragma: no cover
            errs.append(e)

    ts = [threading.Thread(target=work, args=(i,)) for i in range(6)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs
