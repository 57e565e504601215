"""q8-scale codec (src/codec.cpp:27-94): the C
oracle against the reference (CPU), and the device codec against the oracle
byte for byte (GPU). Cases follow test_formats.cpp:137-186 — lengths 2, 100,
4096, 4097, all-zero, the -32768 lane, truncated blobs — plus large payloads
that span many CTA segments."""
import ctypes as ct

import numpy as np
import pytest
import torch

LENGTHS = [0, 1, 2, 3, 100, 4096, 4097, 65536 * 2 + 7, (1 << 20) + 1]


def _payloads():
    rng = np.random.default_rng(5)
    out = [rng.integers(0, 256, size=n, dtype=np.uint8) for n in LENGTHS]
    out.append(np.zeros(512, np.uint8))
    edge = np.zeros(64, np.uint8)
    edge[0], edge[1] = 0x00, 0x80  # lane -32768: |lane| = 32768
    edge[2], edge[3] = 0xFF, 0x7F  # 32767
    out.append(edge)
    small = (rng.integers(-3, 4, size=1000).astype(np.int16)).view(np.uint8)  # tiny scale, many .5 ties
    out.append(small.copy())
    return out


SPECIAL_SCALES = [1.0, 0.5, 1 / 127, 258.0157480314961, 3.0e-5, 1.0e-30, 7.0e5, 8388608.0, 3.0e38,
                  1.0e-40, 0.0, -0.0, -2.5, float("inf"), float("-inf"), float("nan")]


def _scale_blobs():
    """Blobs carrying every int8 code under arbitrary scale bit patterns."""
    q = np.arange(256, dtype=np.uint8)
    scales = SPECIAL_SCALES + list(np.random.default_rng(11).uniform(0.001, 300.0, size=24))
    n = 2 * q.size + 1
    return scales, [np.concatenate([np.frombuffer(np.uint32(n).tobytes(), np.uint8),
                                    np.frombuffer(np.float32(s).tobytes(), np.uint8), q, [0x5A]]).astype(np.uint8)
                    for s in scales], n


def test_oracle_q8_matches_reference(C, Ref):
    for p in _payloads():
        blob = C.q8_encode(p)
        assert np.array_equal(blob, Ref.q8_encode(p)), p.size
        dec, code = Ref.q8_decode(blob)
        assert code == 0 and np.array_equal(C.q8_decode(blob), dec)
    scales, blobs, _ = _scale_blobs()
    for s, b in zip(scales, blobs):
        dec, code = Ref.q8_decode(b)
        assert code == 0 and np.array_equal(C.q8_decode(b), dec), s


def test_oracle_q8_golden(C):
    import hashlib
    import json
    import os
    with open(os.path.join(os.path.dirname(__file__), "golden", "q8.json")) as f:
        g = json.load(f)
    rng = np.random.default_rng(8)
    for case in g["cases"]:
        p = rng.integers(0, 256, size=case["n"], dtype=np.uint8)
        blob = C.q8_encode(p)
        assert hashlib.sha256(blob.tobytes()).hexdigest() == case["blob_sha256"]
        assert hashlib.sha256(C.q8_decode(blob).tobytes()).hexdigest() == case["decoded_sha256"]


def test_oracle_q8_bounds_and_corruption(C):
    """test_formats.cpp:137-186: size ratio, per-lane error bound, raw odd tail,
    exact zeros, truncated / over-long blobs rejected."""
    rng = np.random.default_rng(5)
    for n in (2, 100, 4096, 4097):
        p = rng.integers(0, 256, size=n, dtype=np.uint8)
        blob = C.q8_encode(p)
        if n >= 1000:
            assert 0.45 < blob.size / n < 0.55
        d = C.q8_decode(blob)
        lanes_o = p[: n // 2 * 2].view(np.int16).astype(np.int64)
        lanes_r = d[: n // 2 * 2].view(np.int16).astype(np.int64)
        scale = np.abs(lanes_o).max() / 127.0
        assert np.all(np.abs(lanes_o - lanes_r) <= scale / 2 + 1)
        if n % 2:
            assert d[-1] == p[-1]
    z = np.zeros(512, np.uint8)
    assert np.array_equal(C.q8_decode(C.q8_encode(z)), z)
    blob = C.q8_encode(np.zeros(100, np.uint8))
    assert C.q8_decode(blob[:-3]) is None and C.q8_decode(blob[:3]) is None


@pytest.mark.gpu
def test_device_q8_matches_oracle(tkv, C):
    from paper_2510_09665_b200.api import q8_decode, q8_encode
    ps = [p for p in _payloads() if p.size > 0]
    dev = [torch.from_numpy(p.copy()).cuda() for p in ps]
    blobs = q8_encode(dev)
    for p, b in zip(ps, blobs):
        assert np.array_equal(b.cpu().numpy(), C.q8_encode(p)), p.size
    back = q8_decode(blobs, [p.size for p in ps])
    for p, b, d in zip(ps, blobs, back):
        assert np.array_equal(d.cpu().numpy(), C.q8_decode(C.q8_encode(p))), p.size


@pytest.mark.gpu
@pytest.mark.parametrize("maxabs", [1, 2, 3, 5, 127, 128, 254, 255, 1000, 4097, 12345, 32767, 32768])
def test_device_q8_encode_every_lane(tkv, C, maxabs):
    """Every lane value in [-maxabs, maxabs] (including the exact .5 ties the
    scale produces) quantises to the reference's byte: the device's integer
    rounding against the oracle's double division."""
    from paper_2510_09665_b200.api import q8_decode, q8_encode
    rng = np.random.default_rng(maxabs)
    lanes = np.arange(-maxabs, min(maxabs, 32767) + 1, dtype=np.int64)
    lanes = np.concatenate([lanes, [-maxabs if maxabs == 32768 else maxabs]])
    rng.shuffle(lanes)
    p = lanes.astype(np.int16).view(np.uint8)
    blob = q8_encode([torch.from_numpy(p.copy()).cuda()])[0].cpu().numpy()
    assert np.array_equal(blob, C.q8_encode(p))
    back = q8_decode([torch.from_numpy(blob.copy()).cuda()], [p.size])[0].cpu().numpy()
    assert np.array_equal(back, C.q8_decode(blob))


@pytest.mark.gpu
def test_device_q8_decode_any_scale_bits(tkv, C):
    """Decode takes the scale from the blob: every int8 code under scales that
    are normal, tiny, huge, subnormal, zero, negative, infinite and NaN equals
    the reference's double formula."""
    from paper_2510_09665_b200.api import q8_decode
    scales, blobs, n = _scale_blobs()
    outs = q8_decode([torch.from_numpy(b.copy()).cuda() for b in blobs], [n] * len(blobs))
    for s, b, o in zip(scales, blobs, outs):
        assert np.array_equal(o.cpu().numpy(), C.q8_decode(b)), s


@pytest.mark.gpu
def test_device_q8_encode_batch_pipeline(tkv, C):
    """A batch that exercises the single-pass encode's item pipeline: several
    multi-MiB items (absmax of item p overlapped with the quantise of item
    p - 1), ragged and odd lengths, an empty item, and payloads / blobs at
    offsets that break the 32-byte vector path (scalar fallback inside the
    same launch). Every blob byte equals the oracle's."""
    from paper_2510_09665_b200.api import q8_encode
    rng = np.random.default_rng(77)
    sizes = [32 << 20, (3 << 20) + 6, (1 << 20) + 1, 0, 2, (5 << 20) + 32, 4096 + 3, 8 << 20]
    offsets = [0, 0, 0, 0, 0, 2, 6, 0]  # bytes into a larger allocation: unaligned src
    srcs, host = [], []
    for n, off in zip(sizes, offsets):
        lanes = np.clip(rng.normal(0, 2500 + n % 7000, size=(n + off + 1) // 2 + 1), -32768, 32767).astype(np.int16)
        buf = lanes.view(np.uint8)[: n + off].copy()
        if n >= 2:
            pos = off + ((n // 3) & ~1)
            buf[pos:pos + 2] = [0x00, 0x80]  # one -32768 lane
        host.append(buf[off:])
        srcs.append(torch.from_numpy(buf).cuda()[off:])
    blobs = q8_encode(srcs)
    for n, p, b in zip(sizes, host, blobs):
        assert np.array_equal(b.cpu().numpy(), C.q8_encode(p)), n


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["twopass", "fused"])
def test_q8_encode_variant_subprocess(mode):
    """Both encodes on every shape: the batch shape picks the single-pass
    (fused) encode only for several items of >= 24 MiB, so the encode parity
    tests run again in child processes with TKV_Q8_ENCODE=twopass and
    TKV_Q8_ENCODE=fused (read once per process) forcing one of them."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, TKV_Q8_ENCODE=mode)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu",
                        "tests/test_codec.py::test_device_q8_matches_oracle",
                        "tests/test_codec.py::test_device_q8_encode_batch_pipeline",
                        "tests/test_codec.py::test_device_q8_encode_every_lane",
                        "tests/test_codec.py::test_device_q8_encode_every_lane_vector_path",
                        "tests/test_codec.py::test_device_q8_encode_concurrent_streams"],
                       cwd=root, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


@pytest.mark.gpu
@pytest.mark.parametrize("maxabs", [1, 2, 127, 254, 508, 1000, 12345, 32768])
def test_device_q8_encode_every_lane_vector_path(tkv, C, maxabs):
    """Every lane value in [-maxabs, maxabs], tiled to >= 1 MiB so the
    encode's 32-byte vector path (not only its scalar tail) meets them:
    power-of-two scales (maxabs 127 / 254 / 508: an exact reciprocal, the
    tie case that needs the reciprocal bumped above 1/scale) and the exact
    .5 ties of tiny scales."""
    from paper_2510_09665_b200.api import q8_encode
    lanes = np.arange(-maxabs, min(maxabs, 32767) + 1, dtype=np.int64)
    lanes = np.concatenate([lanes, [-maxabs if maxabs == 32768 else maxabs]])
    reps = max(1, (1 << 19) // lanes.size + 1)
    rng = np.random.default_rng(maxabs + 1)
    tiled = np.tile(lanes, reps)
    rng.shuffle(tiled)
    p = tiled.astype(np.int16).view(np.uint8)
    blob = q8_encode([torch.from_numpy(p.copy()).cuda()])[0].cpu().numpy()
    assert np.array_equal(blob, C.q8_encode(p))


@pytest.mark.gpu
def test_device_q8_encode_concurrent_streams(tkv, C):
    """Encodes issued back to back on two streams with no synchronisation in
    between (each with its own scratch: the single-pass encode's per-item
    counters live there) both produce the oracle's bytes."""
    from paper_2510_09665_b200._lib import CodecItemC, check, lib, u32p
    rng = np.random.default_rng(31)
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    jobs = []
    for k in range(2):
        ps = [np.clip(rng.normal(0, 900 * (k + 1), size=(3 << 19) + 17 * k), -32768, 32767).astype(np.int16)
              .view(np.uint8).copy() for _ in range(3)]
        src = [torch.from_numpy(p).cuda() for p in ps]
        blobs = [torch.empty(int(lib().tkv_q8_blob_bytes(p.size)), dtype=torch.uint8, device="cuda") for p in ps]
        items = (CodecItemC * 3)(*[CodecItemC(s.data_ptr(), b.data_ptr(), p.size) for s, b, p in zip(src, blobs, ps)])
        seg = np.zeros(4, np.uint32)
        check(lib().tkv_codec_plan(ct.cast(items, ct.c_void_p), 3, seg.ctypes.data_as(u32p)))
        d_items = torch.frombuffer(bytearray(bytes(items)), dtype=torch.uint8).cuda()
        d_seg = torch.from_numpy(seg.view(np.int32)).cuda()
        scratch = torch.zeros(int(lib().tkv_q8_encode_scratch_bytes(3)) // 4, dtype=torch.int32, device="cuda")
        jobs.append((ps, src, blobs, d_items, d_seg, int(seg[-1]), scratch))
    torch.cuda.synchronize()
    for (ps, src, blobs, d_items, d_seg, segs, scratch), s in zip(jobs, streams):
        check(lib().tkv_q8_encode(d_items.data_ptr(), d_seg.data_ptr(), 3, segs, scratch.data_ptr(), s.cuda_stream))
    torch.cuda.synchronize()
    for ps, _, blobs, *_ in jobs:
        for p, b in zip(ps, blobs):
            assert np.array_equal(b.cpu().numpy(), C.q8_encode(p))
