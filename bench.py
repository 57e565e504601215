"""KV store+retrieve benchmark (BASELINE.json metric) for the B200 path.

Workload (BASELINE.json configs[2], "Llama-3.1-70B-shaped KV (80 layers,
8 KV heads) TP=N head-sharded store/retrieve at 1/2/4/8 GPUs"): one prompt of
32,768 tokens, chunk 256, page 16. Its first 16,384 tokens (64 chunks) are in
the pinned host tier (prefix hit); the last 16,384 are new. One step is one
scheduling iteration of the reference call sequence
(sim_engine.cpp:97-162): lookup -> alloc -> update_state_after_alloc ->
build_connector_meta -> start_load_kv -> per layer {wait_load_kv, engine
compute of the new tokens, wait_store_kv(l-1), start_store_kv} -> final
wait_store_kv. So every step RETRIEVES 16,384 tokens x 80 layers and STORES
16,384 tokens x 80 layers (fresh suffix each step; LRU recycles old slots).
Under TP=N each rank moves its own head shard: bpt = 4096 / N bytes per
token-layer (8 KV heads x 128 x 2 (K,V) x 2 B / N).

Reported (one JSON line, rank 0):
  value    device-resident throughput: the same step's bytes with the chunk
           side in HBM (K2 scatter of the prefix + K1 gather of the suffix,
           one launch each for all 80 layers), payload GB/s, whole job.
  e2e      the connector step above through the C-ABI with the pinned host
           tier (H2D/D2H inside the timed region), payload GB/s, whole job.
  roofline K1/K2 kernel: algorithmic HBM bytes (2 x payload) / launch time vs
           MEASURED_PEAKS.json hbm_gbs (fallback 6650); traffic from the
           committed ncu capture; links: PCIe measured in-run per rank.
  cpu_baseline  the unmodified reference Connector (oracle/_ref) on one
           step of the same workload (all 80 layers, the full-model rows: the
           reference has no TP, so at N GPUs it does the whole job), rank 0,
           every N, all host cores.
  parity   the 10 GiB page image after the kernel loop; every suffix chunk
           the timed steps stored that is still in the tier (read from its
           pinned slot by the SMs) against synth; and one more (untimed)
           connector step's page image — all checked word by word on device.
  configs  (N = 1) BASELINE.json configs 1, 2 and 4 through the same C-ABI
           connector (tools/bench_configs.py): e2e GB/s and tokens/s, PCIe
           fractions, device byte verification, the reference beside each.
  pd       (N >= 2) prefill rank r -> decode rank r + N/2 chunk sends over
           NVLink: SM-direct, CE-staged and NCCL send/recv variants, in-run
           peer-copy probes (each pair alone, all pairs at once), and the
           reference's PD CPU work on a bounded sample.

--impl reference runs only the reference CPU path (rank 0): the unmodified
reference Connector on the same step (all layers, full rows), one engine
seeded once and reused across steps, with the same config dict. Inputs (64 +
64 chunks of 5 GiB each at N=1) exceed L2 (126 MB), so no L2 flush is needed
between timed steps.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "KV store+retrieve GB/s & tokens/s at 1/2/4/8 B200 vs HBM/PCIe/NVLink roofline"
TAG = "llama-3.1-70b"


def parse():
    return parse_args_list(None)


def parse_args_list(argv):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--prompt", type=int, default=32768)
    ap.add_argument("--prefix", type=int, default=16384)
    ap.add_argument("--layers", type=int, default=80)
    ap.add_argument("--bpt-full", type=int, default=4096)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-configs", action="store_true", help="skip the configs 1/2/4 object (N=1)")
    ap.add_argument("--load-zero-copy", action="store_true")
    ap.add_argument("--store-zero-copy", action="store_true")
    ap.add_argument("--store-ctas", type=int, default=0)
    ap.add_argument("--staging-depth", type=int, default=2)
    ap.add_argument("--ram-slots", type=int, default=0,
                    help="pinned tier slots (0: prefix + two suffixes, so the timed steps evict)")
    ap.add_argument("--profile-kernels", action="store_true", help="only run the K1/K2 device-resident loop")
    ap.add_argument("--trace", action="store_true", help="host time of every call of one step")
    ap.add_argument("--no-pd", action="store_true", help="skip the N>=2 PD-over-NVLink pairs")
    ap.add_argument("--memo-entries", type=int, default=None, help="K3 prefix memo links (0 = off)")
    ap.add_argument("--sequential", action="store_true",
                    help="one request at a time (no overlap of consecutive steps)")
    return ap.parse_args(argv)


def dist_env():
    """(world, rank, device index). TKV_BENCH_DEVICE pins every rank to one
    device (single-GPU exercise of the multi-rank paths, with
    TKV_DIST_BACKEND=gloo since NCCL refuses two ranks on one GPU)."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("TKV_BENCH_DEVICE", os.environ.get("LOCAL_RANK", "0")))
    return world, rank, local


def bind_to_gpu_numa(local):
    """Restrict this rank to the CPUs NVML reports as local to its GPU, before
    any pinned allocation: the pinned host tier is then first-touched on the
    GPU's own NUMA node and its DMA never crosses the socket interconnect.
    Returns the CPU count in use (no-op where NVML or affinity is missing)."""
    try:
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(local)
        words = pynvml.nvmlDeviceGetCpuAffinity(h, 16)
        cpus = {64 * i + b for i, w in enumerate(words) for b in range(64) if (int(w) >> b) & 1}
        avail = os.sched_getaffinity(0)
        if cpus and cpus & avail and (cpus & avail) != avail:
            os.sched_setaffinity(0, cpus & avail)
    except Exception:
        pass
    return len(os.sched_getaffinity(0))


def backend():
    return os.environ.get("TKV_DIST_BACKEND", "nccl")


def coll_device(dev):
    """Where collective tensors live: the GPU for NCCL, the host for gloo."""
    return dev if backend() == "nccl" else "cpu"


_CTL_GROUP = None  # host-side (gloo) group for the per-step control exchange under NCCL


def agree_loaded(loaded, device):
    """The TP hit-length agreement (one MIN all-reduce per step). Under NCCL it
    runs on a gloo group over host memory: a device tensor would need a small
    copy-engine H2D and D2H every step, and those queue behind the layer's KV
    transfers on the copy engines (the stall the engine's prompt uploads
    avoid with SM copies)."""
    from paper_2510_09665_b200.tp import agree_loaded as agree
    if _CTL_GROUP is not None:
        return agree(loaded, "cpu", group=_CTL_GROUP)
    return agree(loaded, device)


def prompt_tokens(n_prefix, n_suffix, step, vocab=128256):
    import numpy as np
    pre = np.random.default_rng(2510).integers(0, vocab, size=n_prefix, dtype=np.uint32)
    suf = np.random.default_rng(10_000 + step).integers(0, vocab, size=n_suffix, dtype=np.uint32)
    return np.concatenate([pre, suf])


# --------------------------------------------------------------- clocks ----

class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        if os.environ.get("TKV_NO_CLOCKS"):  # diagnostics: run without the sampler
            return self
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            self.proc.wait()

    def summary(self, window=None):
        """Median SM clock and the throttle reasons seen. `window` = (t0, t1)
        wall-clock bounds of the timed region: only samples that arrived in
        it count; when fewer than 3 did (a sub-second region), the nearest
        samples of the same workload around it are added and `in_window`
        says how many were strictly inside."""
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        lines = self.lines
        inside = len(lines)
        if window is not None:
            t0, t1 = window
            picked = [x for x in lines if t0 <= x[0] <= t1]
            inside = len(picked)
            if len(picked) < 3:
                mid = 0.5 * (t0 + t1)
                picked = sorted(lines, key=lambda x: abs(x[0] - mid))[:3]
            lines = picked
        for _, ln in lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm), "in_window": inside}


# ------------------------------------------------------------ reference ----

def config_dict(args, world):
    """The workload both arms report (identical dict: same config)."""
    bpt = args.bpt_full // world
    return {"workload": "c3: Llama-3.1-70B KV, 80 layers, TP=N head-sharded, 32K prompt: "
                        "16K prefix retrieve + 16K suffix store per step",
            "prompt": args.prompt, "prefix": args.prefix, "layers": args.layers, "tp": world, "bpt": bpt,
            "chunk": 256, "page": 16, "parallelism": f"tp{world} head-sharded, no data-path collective",
            "l2": "inputs 10 GiB/N >> 126 MB L2, no flush"}


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


class RefStep:
    """The unmodified reference Connector (oracle/_ref, src/connector.cpp:
    71-392) on the bench step: lookup -> update_state_after_alloc ->
    build_connector_meta -> start_load_kv -> per layer {wait_load_kv,
    wait_store_kv(l-1), start_store_kv} -> final wait_store_kv, timed around
    the connector calls only. One engine is seeded once (the stored prefix)
    and reused: the query's pages stay bound with the suffix KV computed once
    (engine compute, untimed), and after each step the suffix chunks are
    cleared from the tier (untimed) so the next step stores them again. Every
    step therefore retrieves the 16K prefix and stores the 16K suffix, all
    layers, full rows — the B200 step's bytes."""

    def __init__(self, args, n_layers, bpt, threads):
        import oracle
        from oracle import RefEngine
        self.ok = oracle.ref_available()
        if not self.ok:
            return
        n, n_pre = args.prompt, args.prefix
        self.n, self.n_pre, self.L, self.bpt = n, n_pre, n_layers, bpt
        chunks = (n + 255) // 256
        self.e = RefEngine(num_layers=n_layers, bpt=bpt, page_tokens=16, tag=TAG, chunk_size=256,
                           ram_slots=chunks + 8, num_pages=(n // 16 + 16) * n_layers, layerwise=True,
                           staging_budget=1 << 40, io_threads=threads, store_io_threads=threads)
        t0 = time.perf_counter()
        self.e.seed_store(prompt_tokens(n_pre, 0, 0), n_pre)  # the stored prefix (setup)
        self.prompt = prompt_tokens(n_pre, n - n_pre, 0)
        self.q = 1
        assert self.e.bind_pages(self.q, n) == 0
        self.e.compute_range(self.q, self.prompt, n_pre, n)  # engine compute of the new tokens
        self.suffix_keys = oracle.C().chunk_keys(self.prompt, 256, TAG)[n_pre // 256:]
        self.setup_s = time.perf_counter() - t0

    def step(self):
        e, q, n, L = self.e, self.q, self.n, self.L
        t0 = time.perf_counter()
        matched = e.get_num_new_matched_tokens(q, self.prompt)
        assert e.update_state_after_alloc(q, (n + 15) // 16, (matched + 15) // 16) == 0
        m = e.build_connector_meta([(q, self.prompt)])
        assert e.start_load_kv(m) == 0
        for layer in range(L):
            assert e.wait_load_kv(m, layer) == 0
            if layer:
                assert e.wait_store_kv(m, layer - 1) == 0
            assert e.start_store_kv(m) == 0
        assert e.wait_store_kv(m, L - 1) == 0
        t = time.perf_counter() - t0
        loaded = e.loaded_tokens(m, q)
        res = e.store_results(m, q)
        assert loaded == self.n_pre, loaded
        assert len(res) == len(self.suffix_keys) and all(c == 0 for _, c in res), res[:2]
        e.drop_meta(m)
        e.finish_query(q)
        for k in self.suffix_keys:  # the next step stores them again
            e.store_clear(k)
        moved = n * L * self.bpt
        return {"gbps": moved / t / 1e9, "seconds": t, "bytes": moved, "tokens": n}

    def close(self):
        if self.ok:
            self.e.close()


def all_cpus():
    """Every CPU of the host (the reference gets all of them, whatever this
    rank's NUMA binding)."""
    try:
        return set(range(os.cpu_count() or 1))
    except Exception:
        return os.sched_getaffinity(0)


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    try:
        os.sched_setaffinity(0, all_cpus())
    except OSError:
        pass
    threads = len(os.sched_getaffinity(0))
    ref = RefStep(args, args.layers, args.bpt_full, threads)
    if not ref.ok:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libtierkv_ref.so not built"}))
        return
    # Each reference step is the whole workload (about 13 s on 16 cores), so
    # the arm times at most 5 steps after at most 1 warm-up: the run ends in
    # under two minutes whatever --steps / --warmup ask for (the line says
    # how many it timed).
    ref_warmup, ref_steps = min(args.warmup, 1), max(1, min(args.steps, 5))
    vals, secs = [], []
    for i in range(ref_warmup + ref_steps):
        r = ref.step()
        if i >= ref_warmup:
            vals.append(r["gbps"])
            secs.append(r["seconds"])
    ref.close()
    v = statistics.median(vals)
    ms = 1e3 * statistics.median(secs)
    sample = (f"every step the full workload: {args.prompt}-token prompt, {args.prefix}-token stored prefix "
              f"retrieved + {args.prompt - args.prefix} tokens stored, all {args.layers} layers, full rows "
              f"(bpt {args.bpt_full}: the reference has no TP, it does the whole {world}-GPU job); one engine "
              f"seeded once ({ref.setup_s:.1f} s setup, untimed), suffix chunks cleared between steps")
    line = {"metric": METRIC, "value": round(v, 4), "unit": "GB/s", "impl": "reference", "n_gpus": world,
            "steps": ref_steps, "warmup": ref_warmup, "steps_requested": args.steps,
            "warmup_requested": args.warmup, "ms_per_step": round(ms, 3),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u8",
            "data": "synthetic (splitmix64 KV from seeded tokens)", "config": config_dict(args, world),
            "tokens_per_s": round(args.prompt / (ms / 1e3), 1),
            "cpu_baseline": {"value": round(v, 4), "unit": "GB/s", "cores": threads, "cpu": cpu_model(),
                             "kind": "reference", "sample": sample},
            "e2e": {"value": round(v, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------- b200 ----

def measure_pcie(torch, dev):
    """Best-of-3 pinned 1 GiB copies per direction and both at once (GB/s)."""
    n = 1 << 30
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device=dev)
    d2 = torch.empty(n, dtype=torch.uint8, device=dev)
    s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)

    def timed(fn):
        best = 1e9
        for _ in range(3):
            torch.cuda.synchronize(dev)
            t0 = time.perf_counter()
            fn()
            torch.cuda.synchronize(dev)
            best = min(best, time.perf_counter() - t0)
        return best

    h2d = n / timed(lambda: d.copy_(h, non_blocking=True)) / 1e9
    d2h = n / timed(lambda: h2.copy_(d2, non_blocking=True)) / 1e9

    def both():
        with torch.cuda.stream(s1):
            d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)
    bi = 2 * n / timed(both) / 1e9
    del h, h2, d, d2
    return {"h2d_gbps": round(h2d, 2), "d2h_gbps": round(d2h, 2), "bidir_gbps": round(bi, 2)}


class B200Bench:
    def __init__(self, args, world, rank, local):
        import numpy as np
        import torch
        from paper_2510_09665_b200.api import Engine
        self.np, self.torch = np, torch
        self.args = args
        self.dev = torch.device(f"cuda:{local}")
        torch.cuda.set_device(self.dev)
        self.world, self.rank = world, rank
        self.bpt = args.bpt_full // world
        self.L = args.layers
        self.n, self.n_pre = args.prompt, args.prefix
        chunks = (self.n + 255) // 256
        self.stream = torch.cuda.Stream(self.dev)
        # Two requests in flight (pipelined schedule): pages for both, and pinned
        # slots for exactly the prefix plus two suffixes: when request k+1
        # reserves, request k's suffix is still being written (not evictable)
        # and request k-1's is committed, so the LRU evicts k-1's suffix, 64
        # consecutive slots (one pitched copy per layer; spare slots would
        # float and split every later store batch into two runs).
        pages = 2 * (self.n // 16 + 16) * self.L
        suffix_chunks = (self.n - self.n_pre + 255) // 256
        self.e = Engine(num_layers=self.L, bpt=self.bpt, page_tokens=16, tag=TAG, chunk_size=256,
                        ram_slots=args.ram_slots or chunks + suffix_chunks, num_pages=pages, layerwise=True,
                        staging_budget=1 << 34, staging_depth=args.staging_depth,
                        load_zero_copy=args.load_zero_copy, store_zero_copy=args.store_zero_copy,
                        store_ctas=args.store_ctas, device=local,
                        stream=self.stream, memo_entries=args.memo_entries,
                        shard_offset=rank * self.bpt)  # this rank's heads: its slice of every row
        self.qid = 100

    def store_prefix(self):
        """Setup: cold prefill of the 16K prefix through the connector."""
        e = self.e
        if self.n_pre == 0:
            return
        pre = prompt_tokens(self.n_pre, 0, 0)
        q = 1
        assert e.get_num_new_matched_tokens(q, pre) == 0
        e.bind_pages(q, len(pre))
        e.update_state_after_alloc(q, (len(pre) + 15) // 16, 0)
        m = e.build_connector_meta([(q, pre)])
        assert e.start_load_kv(m) == 0
        for layer in range(self.L):
            e.wait_load_kv(m, layer)
            e.compute_range(q, pre, 0, len(pre), layers=(layer, layer + 1))
            if layer:
                e.wait_store_kv(m, layer - 1)
            assert e.start_store_kv(m) == 0
        assert e.wait_store_kv(m, self.L - 1) == 0
        assert all(c == 0 for _, c in e.store_results(m, q))
        e.drop_meta(m)
        e.finish_query(q)
        e.release_query(q)

    def lookup(self, k):
        """Scheduler-side lookup of request k (K3 keys + LPM)."""
        prompt = prompt_tokens(self.n_pre, self.n - self.n_pre, k + 1)
        q = self.qid = self.qid + 1
        matched = self.e.get_num_new_matched_tokens(q, prompt)
        assert matched == min(self.n_pre, self.n - 1), matched
        return q, prompt, matched

    def verified_step(self, k):
        """One untimed step through the connector whose retrieved prefix and
        computed suffix are then checked word by word on the device against
        synth (the full-size e2e parity property)."""
        e, L, n = self.e, self.L, self.n
        q, prompt, matched = self.lookup(k)
        assert e.bind_pages(q, n) == 0
        assert e.update_state_after_alloc(q, (n + 15) // 16, (matched + 15) // 16) == 0
        m = e.build_connector_meta([(q, prompt)])
        assert e.start_load_kv(m) == 0
        loaded = e.loaded_tokens(m, q)
        for layer in range(L):
            e.wait_load_kv(m, layer)
            e.compute_range(q, prompt, loaded, n, layers=(layer, layer + 1))
            if layer:
                e.wait_store_kv(m, layer - 1)
            assert e.start_store_kv(m) == 0
        assert e.wait_store_kv(m, L - 1) == 0
        mism = e.verify_range(q, prompt, 0, n)
        e.drop_meta(m)
        e.finish_query(q)
        e.release_query(q)
        return mism, loaded

    def step(self, k, looked_up=None, next_k=None):
        """One scheduling iteration: retrieve the prefix, store the new suffix.

        `looked_up` is request k's lookup if the scheduler already did it;
        with `next_k` the lookup of the next request is issued while this
        step's layers transfer (a serving scheduler's overlap) and returned.
        """
        e, L, n = self.e, self.L, self.n
        q, prompt, matched = looked_up if looked_up is not None else self.lookup(k)
        assert e.bind_pages(q, n) == 0
        assert e.update_state_after_alloc(q, (n + 15) // 16, (matched + 15) // 16) == 0
        m = e.build_connector_meta([(q, prompt)])
        assert e.start_load_kv(m) == 0
        loaded = e.loaded_tokens(m, q)
        for layer in range(L):
            e.wait_load_kv(m, layer)
            e.compute_range(q, prompt, loaded, n, layers=(layer, layer + 1))
            if layer:
                e.wait_store_kv(m, layer - 1)
            assert e.start_store_kv(m) == 0
        nxt = self.lookup(next_k) if next_k is not None else None
        assert e.wait_store_kv(m, L - 1) == 0
        res = e.store_results(m, q)
        assert len(res) == (n - self.n_pre + 255) // 256 and all(c == 0 for _, c in res), res[:2]
        assert loaded == matched
        e.drop_meta(m)
        e.finish_query(q)
        e.release_query(q)
        return loaded, n - self.n_pre, nxt

    def begin(self, looked_up):
        """Enqueue one request's whole step (loads, per-layer compute, stores)."""
        e, L, n = self.e, self.L, self.n
        q, prompt, matched = looked_up
        assert e.bind_pages(q, n) == 0
        assert e.update_state_after_alloc(q, (n + 15) // 16, (matched + 15) // 16) == 0
        m = e.build_connector_meta([(q, prompt)])
        assert e.start_load_kv(m) == 0
        loaded = e.loaded_tokens(m, q)
        if self.world > 1:  # one hit length for the TP forward pass: MIN over ranks (the TP exchange)
            loaded = agree_loaded({q: loaded}, coll_device(self.dev))[q]
        assert loaded == matched
        for layer in range(L):
            e.wait_load_kv(m, layer)
            e.compute_range(q, prompt, loaded, n, layers=(layer, layer + 1))
            if layer:
                e.wait_store_kv(m, layer - 1)
            assert e.start_store_kv(m) == 0
        return q, m, loaded

    def end(self, state):
        """Final store wait and cleanup of a begun step (no device-wide sync)."""
        e = self.e
        q, m, loaded = state
        assert e.wait_store_kv(m, self.L - 1) == 0
        res = e.store_results(m, q)
        assert len(res) == (self.n - self.n_pre + 255) // 256 and all(c == 0 for _, c in res), res[:2]
        if getattr(self, "_pipe_ref", None) is not None:
            o = e.origin_since(m, self._pipe_ref)
            tl = e.timeline(m) + o
            # per step: first/last H2D done, first/last D2H done (ms on one axis)
            self._pipe_tl.append({"origin": round(o, 2), "h2d": [round(float(tl[0, 0]), 2), round(float(tl[-1, 0]), 2)],
                                  "d2h": [round(float(tl[0, 4]), 2), round(float(tl[-1, 4]), 2)],
                                  "layer_ms_h2d": round(float(self.np.median(self.np.diff(tl[:, 0]))), 3),
                                  "layer_ms_d2h": round(float(self.np.median(self.np.diff(tl[:, 4]))), 3)})
        e.drop_meta(m)
        e.finish_query(q)
        e.release_query(q, sync=False)
        return loaded, self.n - self.n_pre

    def run_pipelined(self, ks):
        """Serving-style schedule: request k+1 is looked up and enqueued while
        request k transfers, then k's final store wait returns. Each request
        still does the full reference call sequence; only the batches overlap."""
        tr = [] if os.environ.get("TKV_TRACE_PIPE") else None
        T0 = time.perf_counter()
        if tr is not None:
            self._pipe_ref = self.torch.cuda.Event(enable_timing=True)
            self._pipe_ref.record(self.stream)
            self._pipe_tl = []

        def mark(what):
            if tr is not None:
                tr.append((what, round(1e3 * (time.perf_counter() - T0), 2)))
        st = self.begin(self.lookup(ks[0]))
        out = None
        for i in range(len(ks)):
            nxt = None
            if i + 1 < len(ks):
                mark(f"lookup{i + 1}")
                lk = self.lookup(ks[i + 1])
                mark(f"begin{i + 1}")
                nxt = self.begin(lk)
            mark(f"end{i}")
            out = self.end(st)
            mark(f"ended{i}")
            st = nxt
        if tr is not None:
            print(json.dumps({"pipe_trace_ms": tr, "device_ms": self._pipe_tl}), file=sys.stderr, flush=True)
            self._pipe_ref = None
        return out

    def trace_step(self, k):
        """One step with the host time of every connector call (diagnosis)."""
        e, L, n = self.e, self.L, self.n
        prompt = prompt_tokens(self.n_pre, n - self.n_pre, k + 1)
        q = self.qid = self.qid + 1
        log = []

        def t(name, fn):
            t0 = time.perf_counter()
            r = fn()
            log.append((name, round(1e3 * (time.perf_counter() - t0), 3)))
            return r
        self.torch.cuda.synchronize()
        T0 = time.perf_counter()
        matched = t("lookup", lambda: e.get_num_new_matched_tokens(q, prompt))
        t("bind", lambda: e.bind_pages(q, n))
        t("update", lambda: e.update_state_after_alloc(q, (n + 15) // 16, (matched + 15) // 16))
        m = t("meta", lambda: e.build_connector_meta([(q, prompt)]))
        t("start_load", lambda: e.start_load_kv(m))
        loaded = e.loaded_tokens(m, q)
        for layer in range(L):
            t(f"wait_load{layer}", lambda: e.wait_load_kv(m, layer))
            t(f"compute{layer}", lambda: e.compute_range(q, prompt, loaded, n, layers=(layer, layer + 1)))
            if layer:
                t(f"wait_store{layer - 1}", lambda: e.wait_store_kv(m, layer - 1))
            t(f"start_store{layer}", lambda: e.start_store_kv(m))
        t("final_wait", lambda: e.wait_store_kv(m, L - 1))
        total = 1e3 * (time.perf_counter() - T0)
        tl = e.timeline(m)
        e.drop_meta(m)
        e.finish_query(q)
        e.release_query(q)
        slow = sorted(log, key=lambda x: -x[1])[:12]
        pick = [0, 1, 2, 10, 40, L - 2, L - 1]
        return {"total_ms": round(total, 2), "slowest": slow,
                "timeline_ms[layer]=[h2d,load,compute,gathered,d2h]":
                    {int(i): [round(float(x), 2) for x in tl[i]] for i in pick if i < L},
                "sum_start_store": round(sum(v for k_, v in log if k_.startswith("start_store")), 2),
                "sum_compute": round(sum(v for k_, v in log if k_.startswith("compute")), 2)}

    def step_bytes(self):
        return (self.n_pre + (self.n - self.n_pre)) * self.L * self.bpt

    def verify_stored_steps(self, ks):
        """Every suffix chunk that the steps `ks` stored and the tier still
        holds, read from its pinned slot by the SMs and compared word by word
        with synth of that step's tokens (this rank's row slice). Returns
        (mismatching words, chunks verified, chunks no longer present)."""
        from paper_2510_09665_b200.api import chunk_keys
        mism = verified = gone = 0
        first = self.n_pre // 256
        for k in ks:
            prompt = prompt_tokens(self.n_pre, self.n - self.n_pre, k + 1)
            keys = chunk_keys(prompt, 256, TAG)
            for i in range(first, len(keys)):
                r = self.e.verify_stored(keys[i], prompt, 256 * i, shard_offset=self.rank * self.bpt)
                if r is None:
                    gone += 1
                else:
                    mism += r
                    verified += 1
        return mism, verified, gone


def kernel_loop(bench, steps, warmup):
    """value: device-resident K2 (prefix) + K1 (suffix), all layers per launch."""
    import ctypes as ct
    import numpy as np
    import torch
    from paper_2510_09665_b200.api import XferDescC, plan_tiles
    from paper_2510_09665_b200._lib import check, lib
    e, L, bpt, n, n_pre = bench.e, bench.L, bench.bpt, bench.n, bench.n_pre
    q = 7
    prompt = prompt_tokens(n_pre, n - n_pre, 0)
    assert e.bind_pages(q, n) == 0
    e.compute_range(q, prompt, 0, n)
    table, stride = e.device_table(q)
    torch.cuda.synchronize()
    chunk_b = L * 256 * bpt
    n_chunks = (n + 255) // 256
    hbm = torch.empty(n_chunks * chunk_b, dtype=torch.uint8, device=bench.dev)

    def descs(lo, hi):
        out = []
        for c in range(lo, hi):
            s = c * 256
            d = XferDescC(chunk=hbm.data_ptr() + c * chunk_b, layer_stride=256 * bpt, table_dev=table,
                          table_stride=stride, first_page=s // 16, n_tokens=min(256, n - s))
            out.append(d)
        return out

    pre_d, suf_d = descs(0, n_pre // 256), descs(n_pre // 256, n_chunks)
    page_bytes = 16 * bpt

    def upload(ds):
        if not ds:
            return None
        tb, ppt = plan_tiles(ds, 16, page_bytes, L)
        arr = (XferDescC * len(ds))(*ds)
        dd = torch.frombuffer(bytearray(bytes(arr)), dtype=torch.uint8).to(bench.dev)
        dt = torch.from_numpy(tb.view(np.int32)).to(bench.dev)
        ao = 0
        for d in ds:
            ao |= d.chunk | d.layer_stride
        return dd, dt, int(tb[-1]), ppt, ao

    P, S = upload(pre_d), upload(suf_d)
    layout = e.layout()
    stream = bench.stream
    lib_ = lib()

    def scatter():
        if P:
            check(lib_.tkv_scatter_layers(ct.byref(layout), P[0].data_ptr(), P[1].data_ptr(), len(pre_d), P[2], 0,
                                          L, P[3], P[4], 0, stream.cuda_stream))

    def gather():
        if S:
            check(lib_.tkv_gather_layers(ct.byref(layout), S[0].data_ptr(), S[1].data_ptr(), len(suf_d), S[2], 0, L,
                                         S[3], S[4], 0, stream.cuda_stream))

    # Seed the prefix chunk buffers with the right bytes (K1 gather of the
    # computed pages), so the timed scatter moves real KV.
    if P:
        check(lib_.tkv_gather_layers(ct.byref(layout), P[0].data_ptr(), P[1].data_ptr(), len(pre_d), P[2], 0, L,
                                     P[3], P[4], 0, stream.cuda_stream))
    with torch.cuda.stream(stream):
        for _ in range(warmup):
            scatter()
            gather()
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3 * steps + 1)]
        launches0 = lib_.tkv_launch_count()
        ev[0].record(stream)
        for i in range(steps):
            scatter()
            ev[3 * i + 1].record(stream)
            gather()
            ev[3 * i + 2].record(stream)
            ev[3 * i + 3].record(stream)
        torch.cuda.synchronize()
        launches = lib_.tkv_launch_count() - launches0
    t_sc = [ev[3 * i].elapsed_time(ev[3 * i + 1]) for i in range(steps)]
    t_ga = [ev[3 * i + 1].elapsed_time(ev[3 * i + 2]) for i in range(steps)]
    total_ms = ev[0].elapsed_time(ev[3 * steps])
    mism = e.verify_range(q, prompt, 0, n)  # scatter rewrote the prefix pages with the same bytes
    e.release_query(q)
    del hbm
    torch.cuda.empty_cache()
    pre_bytes = n_pre * L * bpt
    suf_bytes = (n - n_pre) * L * bpt
    return {"total_ms": total_ms, "scatter_ms": statistics.median(t_sc), "gather_ms": statistics.median(t_ga),
            "pre_bytes": pre_bytes, "suf_bytes": suf_bytes, "launches": launches, "mismatch_words": mism}


def run_pd_pairs(args, world, rank, local):
    """Config 5 (N >= 2): prefill ranks [0, N/2) send a 32K-token prompt's KV
    (70B, TP = N/2 head shards) to decode ranks r + N/2 (run_pd's transfer,
    src/sim_engine.cpp:374-472, at chunk granularity). Every rank runs the
    same phases (barriers and NCCL calls are collective):
      1. CE-staged: K1 into local staging, copy-engine peer copies per group;
      2. NCCL: K1 into local staging, ncclSend / ncclRecv of the payload
         (one batch_isend_irecv group per pair; NCCL backend only);
      3. SM-direct: K1 gathers straight into the decoder's landing buffer
         (CUDA IPC mapping: NVLink writes by the SMs) — last, so the landed
         bytes the decoder verifies come from it;
      4. link probes: one plain copy-engine peer copy of 1 GiB per pair, all
         pairs at once and each pair alone;
      5. ordinals over the process group; the decoder checks the PdStaging
         contract (out of order + a duplicate), lands with one K2 and
         verifies every landed byte on device.
    Returns every rank's result dict (rank 0 aggregates)."""
    import ctypes as ct

    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2510_09665_b200._lib import check, lib
    from paper_2510_09665_b200.api import Engine, PdRecordC, PdStaging, pd_land, pd_send, pd_send_staged
    half = world // 2
    tp = half
    bpt = args.bpt_full // tp
    n, L = args.prompt, args.layers
    chunks = (n + 255) // 256
    stride = L * 256 * bpt
    dev = torch.device(f"cuda:{local}")
    prefill = rank < half
    peer = rank + half if prefill else rank - half
    e = Engine(num_layers=L, bpt=bpt, page_tokens=16, tag=TAG, chunk_size=256, ram_slots=2,
               num_pages=(n // 16 + 16) * L, device=local, shard_offset=(rank % half) * bpt)
    prompt = prompt_tokens(n, 0, 999)
    qid = 5000
    payload = n * L * bpt  # bytes per pair
    landing = None
    handle = np.zeros(64, np.uint8)
    offset = ct.c_uint64(0)
    if not prefill:
        landing = torch.empty(chunks * stride, dtype=torch.uint8, device=dev)
        check(lib().tkv_ipc_get_handle(landing.data_ptr(), handle.ctypes.data_as(ct.POINTER(ct.c_uint8)),
                                       ct.byref(offset)))
    handles = [None] * world
    dist.all_gather_object(handles, (handle.tobytes(), offset.value))
    result = {}
    staging = peer_ptr = None
    if prefill:
        peer_ptr = ct.c_void_p()
        h = np.frombuffer(handles[peer][0], np.uint8).copy()
        peer_off = handles[peer][1]
        check(lib().tkv_ipc_open_handle(h.ctypes.data_as(ct.POINTER(ct.c_uint8)), peer_off, ct.byref(peer_ptr)))
        e.bind_pages(qid, n)
        e.compute_range(qid, prompt, 0, n)  # prefill compute stand-in
        staging = torch.empty(chunks * stride, dtype=torch.uint8, device=dev)
        torch.cuda.synchronize(dev)
    reps = 1 + args.steps

    def timed(fn):
        """min over reps of one synchronizing call (the first is a warm-up)."""
        times, out = [], None
        for it in range(reps):
            torch.cuda.synchronize(dev)
            t0 = time.perf_counter()
            out = fn()
            torch.cuda.synchronize(dev)
            if it:
                times.append(time.perf_counter() - t0)
        return min(times), out

    # 1. CE-staged (prefill ranks only; each send returns after its bytes landed)
    if prefill:
        result["t_ce"], _ = timed(lambda: pd_send_staged(e, qid, n, peer_ptr.value, stride, staging.data_ptr()))
    dist.barrier()
    # 2. NCCL send/recv of the gathered payload
    nccl = backend() == "nccl"
    if nccl:
        recv_t = landing[:payload] if landing is not None else None
        if prefill:
            def nccl_send():
                recs = pd_send(e, qid, n, staging.data_ptr(), stride)  # K1 into local staging
                # staging holds chunk i at i * stride; the tail chunks are
                # contiguous up to the last record's end
                nbytes = (len(recs) - 1) * stride + recs[-1].bytes
                for w in dist.batch_isend_irecv([dist.P2POp(dist.isend, staging[:nbytes], peer)]):
                    w.wait()
            result["t_nccl"], _ = timed(nccl_send)
        else:
            nbytes = (chunks - 1) * stride + (n - 256 * (chunks - 1)) * L * bpt
            recv_t = landing[:nbytes]

            def nccl_recv():
                for w in dist.batch_isend_irecv([dist.P2POp(dist.irecv, recv_t, peer)]):
                    w.wait()
            timed(nccl_recv)
    dist.barrier()
    # 3a. layer-streamed at page granularity: one K1 per layer into 16-token
    #     window records (run_pd's PdGranularity::page), as a prefill would
    #     issue it layer by layer (here without the compute in between)
    if prefill:
        from paper_2510_09665_b200.api import PdLayerSender

        def streamed():
            snd = PdLayerSender(e, qid, n, 16, peer_ptr.value, L * 16 * bpt)
            for layer in range(L):
                assert snd.layer(layer) == 0
            r = snd.finish()
            snd.close()
            return r
        result["t_layers"], wrecs = timed(streamed)
        assert len(wrecs) == (n + 15) // 16
    dist.barrier()
    # 3. SM-direct (its landed bytes are the ones verified)
    recs = None
    if prefill:
        result["t_sm"], recs = timed(lambda: pd_send(e, qid, n, peer_ptr.value, stride))
    dist.barrier()
    # 4. link probes: a plain CE peer copy of 1 GiB per pair
    probe = min(1 << 30, chunks * stride)

    def raw():
        check(lib().tkv_ce_copy(ct.c_void_p(staging.data_ptr()), ct.c_void_p(peer_ptr.value), probe, None))
        torch.cuda.synchronize(dev)
    best_all = best_alone = 1e9
    for _ in range(3):  # all pairs at once
        dist.barrier()
        if prefill:
            t0 = time.perf_counter()
            raw()
            best_all = min(best_all, time.perf_counter() - t0)
    for p in range(half):  # each pair alone
        for _ in range(3):
            dist.barrier()
            if prefill and rank == p:
                t0 = time.perf_counter()
                raw()
                best_alone = min(best_alone, time.perf_counter() - t0)
    dist.barrier()
    # 5. ordinals, PdStaging contract, land, verify
    if prefill:
        meta = torch.tensor([[r.addr - peer_ptr.value, r.bytes, r.token_count, r.first_token] for r in recs],
                            dtype=torch.int64, device=coll_device(dev))
        dist.send(meta, dst=peer)
        lib().tkv_ipc_close(peer_ptr, peer_off)
        moved = sum(r.bytes for r in recs)
        best = min(result["t_sm"], result["t_ce"], result.get("t_nccl", 1e9))
        result = {"pair": f"{rank}->{peer}", "gbps": moved / best / 1e9, "bytes": moved, "ms": 1e3 * best,
                  "sm_direct_gbps": moved / result["t_sm"] / 1e9, "ce_staged_gbps": moved / result["t_ce"] / 1e9,
                  "layer_streamed_page_gbps": moved / result["t_layers"] / 1e9,
                  "nccl_gbps": moved / result["t_nccl"] / 1e9 if "t_nccl" in result else None,
                  "link_all_pairs_gbps": probe / best_all / 1e9, "link_alone_gbps": probe / best_alone / 1e9}
    else:
        meta = torch.zeros((chunks, 4), dtype=torch.int64, device=coll_device(dev))
        dist.recv(meta, src=peer)
        st = PdStaging()
        assert st.register_query(qid) == 0
        m = meta.cpu().tolist()
        order = list(range(chunks))[::-1] + [0]  # out of order + a duplicate
        for o in order:
            off, nbytes, cnt, first = m[o]
            rec = PdRecordC(addr=landing.data_ptr() + off, bytes=nbytes, token_count=cnt, first_token=first)
            assert st.push(qid, o, o == chunks - 1, rec) == 0
        rc, landed = st.await_(qid)
        assert rc == 0 and len(landed) == chunks
        e.bind_pages(qid, n)
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        pd_land(e, qid, landed)
        torch.cuda.synchronize(dev)
        land_ms = 1e3 * (time.perf_counter() - t0)
        mism = e.verify_range(qid, prompt, 0, n)
        result = {"pair": f"{peer}->{rank}", "land_ms": land_ms, "mismatch_words": mism}
    out = [None] * world
    dist.all_gather_object(out, result)
    e.close()
    del landing, staging
    torch.cuda.empty_cache()
    return out


def reference_pd_gbps(L, bpt, n_chunks=4):
    """CPU work of the reference's PD transfer per chunk (run_pd,
    src/sim_engine.cpp:389-397 and 441-455): LMCK encode of the prefilled
    chunk (payload copy + FNV-1a) and parse on the decoder (FNV check +
    copy), on a bounded sample of chunks of the pair's geometry. TCP is left
    out, so this is the reference's best case."""
    import oracle
    if not oracle.ref_available():
        return None
    import numpy as np
    C, R = oracle.C(), oracle.Ref()
    toks = prompt_tokens(256 * n_chunks, 0, 999)
    seed = C.model_seed(TAG)
    keys = C.chunk_keys(toks, 256, TAG)
    t = 0.0
    for i in range(n_chunks):
        pay = C.synth_chunk(seed, toks, 256 * i, 256, L, bpt)
        t0 = time.perf_counter()
        rec = R.encode_record(TAG, keys[i], 256, L, bpt, pay)
        code, back = R.parse_record(rec, pay.size)
        t += time.perf_counter() - t0
        assert code == 0 and np.array_equal(back, pay)
    moved = n_chunks * 256 * L * bpt
    return {"value": round(moved / t / 1e9, 4), "unit": "GB/s", "cores": 1, "kind": "reference",
            "sample": f"{n_chunks} chunks of {L} layers x 256 tokens x {bpt} B: LMCK encode + parse "
                      f"(run_pd's CPU work, TCP excluded)"}


def ncu_traffic(kernel, algorithmic_bytes, bench):
    """roofline.traffic: DRAM bytes per launch of `kernel` from the committed
    ncu --set full capture (profiles/ncu_traffic.json), when that capture was
    taken on this exact workload; otherwise null."""
    out = {"traffic": None, "algorithmic_bytes": int(algorithmic_bytes)}
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            t = json.load(f)
    except (OSError, ValueError):
        return out
    want = {"prompt": bench.n, "prefix": bench.n_pre, "layers": bench.L, "bpt": bench.bpt}
    k = t.get("kernels", {}).get(kernel)
    if k is None or t.get("config") != want:
        return out
    out["traffic"] = int(k["dram_read"] + k["dram_write"])
    out["traffic_source"] = t.get("source")
    out["traffic_frac_of_algorithmic"] = round(out["traffic"] / algorithmic_bytes, 4)
    return out


def run_b200(args):
    import numpy as np  # noqa: F401
    import torch
    import torch.distributed as dist

    world, rank, local = dist_env()
    bind_to_gpu_numa(local)
    if world > 1:
        if backend() == "nccl":
            torch.cuda.set_device(local)  # NCCL collectives run on the current device
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
            global _CTL_GROUP
            _CTL_GROUP = dist.new_group(backend="gloo")
        else:
            dist.init_process_group(backend())
    # nvidia-smi (NVML init) takes a second or more to come up and perturbs the
    # device while it does: start the clock sampler now, seconds before the
    # timed region; only the samples that arrive inside it are summarised.
    clk = ClockSampler(local).__enter__()
    bench = B200Bench(args, world, rank, local)
    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peaks = json.load(f)
    except OSError:
        pass
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    peak_source = ("MEASURED_PEAKS.json hbm_gbs (copy, read+write)" if "hbm_gbs" in peaks
                   else "fallback 6650 GB/s (B200_PROFILING.md; MEASURED_PEAKS.json absent)")
    pcie = measure_pcie(torch, bench.dev)
    pcie_all = [pcie]
    if world > 1:  # every rank's own link, for the per-GPU and aggregate roofline
        pcie_all = [None] * world
        dist.all_gather_object(pcie_all, pcie)

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=coll_device(bench.dev))
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- value: device-resident kernels
    barrier()
    kr = kernel_loop(bench, args.steps, args.warmup)
    k_ms = max_over_ranks(kr["total_ms"] / args.steps)
    mism_all = kr["mismatch_words"]
    if world > 1:  # every rank's page image, not rank 0's alone
        t = torch.tensor([float(mism_all)], dtype=torch.float64, device=coll_device(bench.dev))
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        mism_all = int(t.item())
    step_bytes_rank = kr["pre_bytes"] + kr["suf_bytes"]
    value = step_bytes_rank * world / (k_ms / 1e3) / 1e9
    if args.profile_kernels:
        clk.__exit__()
        if rank == 0:
            print(json.dumps({"kernels": kr}), flush=True)
        return
    # ---- e2e: the connector step through the C-ABI, pinned host tier
    bench.store_prefix()
    # Warm-up runs the same schedule as the timed region: the pipelined one
    # keeps two requests in flight, and its first steps grow the launch-plan
    # and page-table pools (pinned + device allocations) to that depth.
    if args.sequential or args.trace:
        for k in range(args.warmup):
            bench.step(k)
    elif args.warmup:
        bench.run_pipelined(list(range(args.warmup)))
    if args.trace:
        clk.__exit__()
        if rank == 0:
            print(json.dumps({"trace": bench.trace_step(1000)}), flush=True)
        return
    barrier()
    torch.cuda.synchronize()
    lib_ = bench.e.L
    launches0 = lib_.tkv_launch_count()
    copies0 = bench.e.copy_runs()
    w0 = time.time()
    start = torch.cuda.Event(enable_timing=True)
    end = torch.cuda.Event(enable_timing=True)
    start.record(bench.stream)
    t0 = time.perf_counter()
    if args.sequential:
        nxt = bench.lookup(args.warmup)
        for k in range(args.steps):
            kk = args.warmup + k
            loaded, stored, nxt = bench.step(kk, looked_up=nxt, next_k=kk + 1 if k + 1 < args.steps else None)
    else:
        loaded, stored = bench.run_pipelined([args.warmup + k for k in range(args.steps)])
    torch.cuda.synchronize()
    end.record(bench.stream)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    w1 = time.time()
    time.sleep(0.25)  # let the sampler deliver the samples taken inside the region
    clk.__exit__()
    e2e_launches = lib_.tkv_launch_count() - launches0
    copies1 = bench.e.copy_runs()
    host_pieces, host_copies = copies1[0] - copies0[0], copies1[1] - copies0[1]
    # parity of the timed schedule itself: every suffix chunk the timed steps
    # stored that the tier still holds, read back from its slot on device
    ts_mism, ts_ok, ts_gone = bench.verify_stored_steps([args.warmup + k for k in range(args.steps)])
    e2e_mism, e2e_loaded = bench.verified_step(args.warmup + args.steps)  # untimed parity step
    if world > 1:
        t = torch.tensor([float(e2e_mism), float(ts_mism), float(ts_ok), float(ts_gone)], dtype=torch.float64,
                         device=coll_device(bench.dev))
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        e2e_mism, ts_mism, ts_ok, ts_gone = (int(x) for x in t.tolist())
    e2e_ms = max_over_ranks(start.elapsed_time(end) / args.steps)
    barrier()
    e2e_bytes_rank = (loaded + stored) * bench.L * bench.bpt
    e2e = e2e_bytes_rank * world / (e2e_ms / 1e3) / 1e9
    tokens_per_s = (loaded + stored) / (e2e_ms / 1e3)

    pd = None
    pd_failed = False
    if world >= 2 and world % 2 == 0 and not args.no_pd:
        try:
            res = run_pd_pairs(args, world, rank, local)
            sends = [r for r in res if "gbps" in r]
            lands = [r for r in res if "land_ms" in r]
            agg = sum(r["gbps"] for r in sends)
            mism = sum(r["mismatch_words"] for r in lands)
            nccl = [r["nccl_gbps"] for r in sends]
            pd = {"ok": mism == 0, "pairs": len(sends), "per_pair_gbps": [round(r["gbps"], 1) for r in sends],
                  "sm_direct_gbps": [round(r["sm_direct_gbps"], 1) for r in sends],
                  "ce_staged_gbps": [round(r["ce_staged_gbps"], 1) for r in sends],
                  "layer_streamed_page_gbps": [round(r["layer_streamed_page_gbps"], 1) for r in sends],
                  "nccl_gbps": [round(x, 1) for x in nccl] if all(x is not None for x in nccl) else None,
                  "aggregate_gbps": round(agg, 1), "bytes_per_pair": sends[0]["bytes"],
                  "land_ms": [round(r["land_ms"], 3) for r in lands], "mismatch_words": mism,
                  "link_alone_gbps": [round(r["link_alone_gbps"], 1) for r in sends],
                  "link_all_pairs_gbps": [round(r["link_all_pairs_gbps"], 1) for r in sends],
                  "frac_of_link_alone": round(min(r["gbps"] / r["link_alone_gbps"] for r in sends), 4),
                  "frac_of_link_all_pairs": round(min(r["gbps"] / r["link_all_pairs_gbps"] for r in sends), 4),
                  "link_probe": "in-run copy-engine peer copy of 1 GiB per pair (cudaMemcpyAsync over NVLink), "
                                "best of 3, each pair alone and all pairs at once",
                  "cpu_baseline": (reference_pd_gbps(args.layers, args.bpt_full // (world // 2))
                                   if rank == 0 and not args.no_cpu_baseline else None),
                  "path": "per pair the fastest of: K1 gather straight into the peer decoder's landing buffer "
                          "(CUDA IPC, SM writes over NVLink) | K1 into local staging + copy-engine peer copies "
                          "per 1 GiB group | K1 into local staging + ncclSend/ncclRecv; PdStaging ordinal "
                          "contract, one K2 land, bytes verified on device"}
            pd_failed = mism != 0
        except Exception as ex:  # the headline line still prints; the run then fails (rc 3)
            pd = {"ok": False, "error": repr(ex)[:300]}
            pd_failed = True
    configs = None
    if world == 1 and not args.no_configs:
        bench.e.close()  # its pinned tier and pages are not needed any more
        torch.cuda.empty_cache()
        sys.path.insert(0, os.path.join(ROOT, "tools"))
        import bench_configs
        configs = bench_configs.run_all(pcie, cpu=not args.no_cpu_baseline)
    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        # the reference on one step of the whole job (full rows: it has no TP),
        # on every host core; after every timed region, rank 0 only
        aff = os.sched_getaffinity(0)
        try:
            os.sched_setaffinity(0, all_cpus())
        except OSError:
            pass
        threads = len(os.sched_getaffinity(0))
        ref = RefStep(args, args.layers, args.bpt_full, threads)
        if ref.ok:
            r = ref.step()
            ref.close()
            cpu = {"value": round(r["gbps"], 4), "unit": "GB/s", "cores": threads, "cpu": cpu_model(),
                   "kind": "reference",
                   "sample": f"one step of the same workload: {args.prefix}-token prefix retrieved + "
                             f"{args.prompt - args.prefix} tokens stored, all {args.layers} layers, full rows "
                             f"(bpt {args.bpt_full}, the whole {world}-GPU job), {r['seconds']:.2f} s "
                             f"(setup {ref.setup_s:.1f} s untimed)"}
        try:
            os.sched_setaffinity(0, aff)
        except OSError:
            pass
    if rank != 0:
        return
    dom_ms = max(kr["scatter_ms"], kr["gather_ms"])
    dom = "K2 scatter (prefix, all layers)" if kr["scatter_ms"] >= kr["gather_ms"] else "K1 gather (suffix, all layers)"
    dom_bytes = 2 * (kr["pre_bytes"] if kr["scatter_ms"] >= kr["gather_ms"] else kr["suf_bytes"])
    achieved = dom_bytes / (dom_ms / 1e3) / 1e9
    h2d = bench.n_pre * bench.L * bench.bpt + bench.n * 4 + bench.L * (bench.n // 16) * 4
    d2h = (bench.n - bench.n_pre) * bench.L * bench.bpt + ((bench.n + 255) // 256) * 32
    line = {
        "metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(e2e_ms, 3), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u8", "data": "synthetic (splitmix64 KV from seeded tokens, device-generated)",
        "config": config_dict(args, world),
        "value_kind": "device-resident K2+K1 payload GB/s (chunk side in HBM)",
        "kernel_ms_per_step": round(k_ms, 3),
        "tokens_per_s": round(tokens_per_s, 1),
        "e2e": {"value": round(e2e, 2), "unit": "GB/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "ms_per_step": round(e2e_ms, 3), "wall_ms_per_step": round(1e3 * wall / args.steps, 3),
                "path": "C-ABI connector: K3 lookup, "
                        + ("zero-copy K2 loads" if args.load_zero_copy else "CE pitched H2D + K2 scatter")
                        + ", " + ("K1 zero-copy store" if args.store_zero_copy
                                  else "K1 gather to HBM ring + CE pitched D2H store"),
                "host_tier_pieces": host_pieces, "host_tier_copies": host_copies,
                "host_tier_copy_note": "chunk-layer slices moved by the copy engines in the timed region and "
                                       "the copies issued for them (one cudaMemcpy2DAsync per run of slots "
                                       "at a constant pitch)"},
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": round(achieved, 1), "peak": hbm_peak,
                     "unit": "GB/s", "frac": round(achieved / hbm_peak, 4),
                     **ncu_traffic(dom, dom_bytes, bench), "peak_source": peak_source},
        "links": {"pcie": pcie, "pcie_bidir_per_rank": [p["bidir_gbps"] for p in pcie_all],
                  "pcie_bidir_aggregate": round(sum(p["bidir_gbps"] for p in pcie_all), 2),
                  "e2e_frac_of_pcie_bidir": round(e2e / sum(p["bidir_gbps"] for p in pcie_all), 4)},
        "gpu_launches": int(e2e_launches),
        "kernel_launches_value": int(kr["launches"]),
        "parity": {"value_pages_mismatch_words": mism_all, "ranks_checked": world,
                   "timed_store_mismatch_words": ts_mism, "timed_store_chunks_verified": ts_ok,
                   "timed_store_chunks_evicted": ts_gone,
                   "timed_store_check": "after the timed loop: every suffix chunk the timed steps stored that "
                                        "the tier still holds (LRU evicted the rest), read from its pinned slot "
                                        "by the SMs and compared word by word with synth of that step's tokens",
                   "e2e_pages_mismatch_words": e2e_mism,
                   "e2e_check": f"one more connector step after the timed region: {e2e_loaded}-token prefix "
                                f"retrieved from the pinned tier + {bench.n - e2e_loaded} computed tokens, "
                                f"every page word of all {bench.L} layers against synth on the device"},
        "cpu_baseline": cpu,
        "clocks": clk.summary((w0, w1)),
    }
    if pd is not None:
        line["pd"] = pd
    if configs is not None:
        line["configs"] = configs
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    if pd_failed or ts_mism or e2e_mism or mism_all:
        sys.exit(3)  # a parity or PD failure fails the run (the line above says which)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
