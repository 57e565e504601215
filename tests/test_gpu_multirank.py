"""The N >= 2 bench path, exercised on one GPU: `torchrun --nproc-per-node 2
bench.py` with every rank pinned to cuda:0 (TKV_BENCH_DEVICE=0) over gloo
(NCCL refuses two ranks on one device). Runs the multi-rank code the
driver's scaling run uses — TP head shards per rank, the per-step TP
agreement (MIN of the delivered prefix), max-over-ranks timing, the PD pair
over CUDA IPC (SM-direct and CE-staged sends, link probes, PdStaging, land,
verify) — at a reduced size, and checks every parity counter of the line."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_bench_two_ranks_on_one_gpu():
    env = dict(os.environ, TKV_BENCH_DEVICE="0", TKV_DIST_BACKEND="gloo", TKV_NO_CLOCKS="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus", "2",
           "--steps", "2", "--warmup", "1", "--no-cpu-baseline", "--prompt", "8192", "--prefix", "4096",
           "--layers", "8"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([x for x in r.stdout.splitlines() if x.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["config"]["tp"] == 2 and line["config"]["bpt"] == 2048
    par = line["parity"]
    assert par["ranks_checked"] == 2
    assert par["value_pages_mismatch_words"] == 0 and par["e2e_pages_mismatch_words"] == 0
    assert par["timed_store_mismatch_words"] == 0 and par["timed_store_chunks_verified"] > 0
    pd = line["pd"]
    assert pd["ok"] and pd["pairs"] == 1 and pd["mismatch_words"] == 0, pd
    assert pd["sm_direct_gbps"][0] > 0 and pd["ce_staged_gbps"][0] > 0 and pd["layer_streamed_page_gbps"][0] > 0
    assert pd["nccl_gbps"] is None  # gloo: the NCCL variant runs only under NCCL
    assert pd["link_alone_gbps"][0] > 0 and pd["link_all_pairs_gbps"][0] > 0
    assert line["e2e"]["value"] > 0 and line["gpu_launches"] > 0
