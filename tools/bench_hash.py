"""K3 (chained SHA-256 chunk keys) timing on the B200.

Cases: one 32K-token chain (bench config 3 lookup), 64 chains of 20K tokens
(config 2 batch lookup), one 128K-token document chain (config 4), and
1024 chains of 4K tokens (throughput). Device time by CUDA events around
tkv_hash_chains; the reference chain (OpenSSL SHA-NI, oracle/_ref) is timed
on the host for the same tokens when available. Also checks every digest
against the CPU oracle for the smaller cases.
"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2510_09665_b200.api import ChainDescC, hash_chains  # noqa: E402

TAG = "llama-3.1-70b"


def run_case(name, lens, reps=5, check=False):
    rng = np.random.default_rng(len(lens))
    toks = [rng.integers(0, 128256, size=n, dtype=np.uint32) for n in lens]
    flat = np.concatenate(toks + [np.zeros(4, np.uint32)])
    chains = (ChainDescC * len(lens))()
    off = row = 0
    for i, n in enumerate(lens):
        chains[i].token_off, chains[i].n_tokens, chains[i].out_first = off, n, row
        off += n
        row += (n + 255) // 256
    dt = torch.from_numpy(flat.view(np.int32)).cuda()
    dc = torch.frombuffer(bytearray(bytes(chains)), dtype=torch.uint8).cuda()
    out = torch.zeros(row * 32, dtype=torch.uint8, device="cuda")
    s = torch.cuda.current_stream()
    hash_chains(dt, dc, len(lens), 256, TAG, out)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        hash_chains(dt, dc, len(lens), 256, TAG, out)
        b.record(s)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ms = min(ts)
    tokens = sum(lens)
    res = {"case": name, "chains": len(lens), "chunks": row, "tokens": tokens, "gpu_ms": round(ms, 4),
           "gpu_us_per_chunk_serial": round(1e3 * ms / max(1, row // len(lens)), 3),
           "gpu_mtok_s": round(tokens / ms / 1e3, 2)}
    try:
        import oracle
        if oracle.ref_available():
            R = oracle.Ref()
            n_ref = min(len(lens), 8)
            t0 = time.perf_counter()
            ref = [R.chunk_keys(t, 256, TAG) for t in toks[:n_ref]]
            cpu = time.perf_counter() - t0
            ref_tokens = sum(lens[:n_ref])
            res["ref_cpu_ms_per_chain"] = round(1e3 * cpu / n_ref, 3)
            res["ref_cpu_mtok_s_1core"] = round(ref_tokens / cpu / 1e6, 2)
            if check:
                o = out.cpu().numpy()
                r = 0
                for i in range(n_ref):
                    got = [o[32 * (r + k):32 * (r + k + 1)].tobytes() for k in range(len(ref[i]))]
                    assert got == ref[i], f"{name}: chain {i} differs"
                    r += len(ref[i])
                res["checked_chains"] = n_ref
    except Exception as e:  # reference missing on the box is fine
        res["ref_error"] = str(e)[:80]
    print(json.dumps(res), flush=True)
    return res


if __name__ == "__main__":
    run_case("1x32K (config 3 lookup)", [32768], check=True)
    run_case("64x20K (config 2 batch lookup)", [20480] * 64, check=True)
    run_case("1x128K (config 4 document)", [131072], reps=3, check=True)
    run_case("1024x4K (throughput)", [4096] * 1024, reps=3)
    run_case("4096x4K (throughput)", [4096] * 4096, reps=3)
