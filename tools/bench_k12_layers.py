"""K1/K2 at the launch sizes the connector issues (verdict r01 item 8).

The layerwise connector launches one K2 (load) and one K1 (store) per layer:
16,384 tokens x bpt per launch = 64 MiB at bpt 4096 (TP=1) down to 8 MiB at
bpt 512 (TP=8). This times exactly those one-layer launches back to back on
one stream (CUDA events around each launch), next to the all-layer launch of
bench.py's kernel loop, and reports algorithmic HBM GB/s (2 x payload / time)
against MEASURED_PEAKS.json. Prints one JSON line per (bpt, direction).

    python tools/bench_k12_layers.py [--bpt 4096 2048 1024 512] [--reps 5]
"""
from __future__ import annotations

import argparse
import ctypes as ct
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--bpt", type=int, nargs="+", default=[4096, 2048, 1024, 512])
    ap.add_argument("--tokens", type=int, default=16384)
    ap.add_argument("--layers", type=int, default=80)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--ctas", type=int, default=0)
    ap.add_argument("--affine", action="store_true",
                    help="launch through tkv_*_layers_affine (the connector's one-query form) instead of "
                         "the descriptor-list entry points")
    args = ap.parse_args()
    import numpy as np
    import torch

    from paper_2510_09665_b200._lib import AffinePlanC, check, lib
    from paper_2510_09665_b200.api import Engine, XferDescC, plan_tiles
    peak = 6650.0
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peak = float(json.load(f)["hbm_gbs"])
    except (OSError, KeyError, ValueError):
        pass
    L, n = args.layers, args.tokens
    dev = torch.device("cuda:0")
    stream = torch.cuda.Stream(dev)
    lib_ = lib()
    for bpt in args.bpt:
        e = Engine(num_layers=L, bpt=bpt, page_tokens=16, tag="k12", chunk_size=256, ram_slots=1,
                   num_pages=(n // 16 + 16) * L, device=0, stream=stream)
        q = 1
        prompt = np.arange(n, dtype=np.uint32)
        assert e.bind_pages(q, n) == 0
        e.compute_range(q, prompt, 0, n)
        table, tstride = e.device_table(q)
        torch.cuda.synchronize()
        n_chunks = (n + 255) // 256
        # the connector's staging-ring layout (chunk i's layer slice at
        # i * 256 * bpt), one slot per layer so no launch finds its chunk side
        # in L2 (a worst case: the product's 2-deep ring may partly hit L2)
        slot = n_chunks * 256 * bpt
        ring = torch.empty(L * slot, dtype=torch.uint8, device=dev)
        descs = [XferDescC(chunk=ring.data_ptr() + c * 256 * bpt, layer_stride=slot, table_dev=table,
                           table_stride=tstride, first_page=(c * 256) // 16, n_tokens=256)
                 for c in range(n_chunks)]
        # the connector's plans: one page per tile for one-layer launches (unit
        # kernel), ~64 KiB tiles for all-layer ones; TKV_PAGED_KERNEL=tile
        # forces the tile kernel with its own tiles everywhere (round-1 code)
        unit = os.environ.get("TKV_PAGED_KERNEL") != "tile"
        tb, ppt = plan_tiles(descs, 16, 16 * bpt, 1, 1 if unit else 0)
        tb_all, ppt_all = plan_tiles(descs, 16, 16 * bpt, L)
        arr = (XferDescC * len(descs))(*descs)
        d_desc = torch.frombuffer(bytearray(bytes(arr)), dtype=torch.uint8).to(dev)
        d_tb = torch.from_numpy(tb.view(np.int32)).to(dev)
        d_tb_all = torch.from_numpy(tb_all.view(np.int32)).to(dev)
        tb_one, _ = plan_tiles(descs[:1], 16, 16 * bpt, 1)
        tb_one[-1] = 1  # a single page: the per-launch floor
        d_tb_one = torch.from_numpy(tb_one.view(np.int32)).to(dev)
        ao = 0
        for d in descs:
            ao |= d.chunk | d.layer_stride
        layout = e.layout()
        payload = n * bpt
        aff = AffinePlanC()
        check(lib_.tkv_affine_form(ct.cast(arr, ct.c_void_p), len(descs), 16, ct.byref(aff)))
        affine_fn = {id(lib_.tkv_gather_layers): lib_.tkv_gather_layers_affine,
                     id(lib_.tkv_scatter_layers): lib_.tkv_scatter_layers_affine}

        def launch(fn, layer):
            if args.affine:
                check(affine_fn[id(fn)](ct.byref(layout), ct.byref(aff), layer, 1, args.ctas, stream.cuda_stream))
                return
            check(fn(ct.byref(layout), d_desc.data_ptr(), d_tb.data_ptr(), len(descs), int(tb[-1]), layer, 1,
                     ppt, ao, args.ctas, stream.cuda_stream))

        def timed(fn, reps=20):
            with torch.cuda.stream(stream):
                for _ in range(3):
                    fn()
                ev = [torch.cuda.Event(enable_timing=True) for _ in range(reps + 1)]
                torch.cuda._sleep(8_000_000)  # host enqueues ahead (see above)
                ev[0].record(stream)
                for i in range(reps):
                    fn()
                    ev[i + 1].record(stream)
                torch.cuda.synchronize()
            return statistics.median(ev[i].elapsed_time(ev[i + 1]) for i in range(reps))

        # K1 first (reads the computed pages), then K2 (overwrites them with
        # the ring's last layer: timing only, parity is tested elsewhere)
        for name, fn in (("K1 gather", lib_.tkv_gather_layers), ("K2 scatter", lib_.tkv_scatter_layers)):
            with torch.cuda.stream(stream):
                for layer in range(L):  # warm-up pass
                    launch(fn, layer)
                torch.cuda.synchronize()
                times = []
                for _ in range(args.reps):
                    ev = [torch.cuda.Event(enable_timing=True) for _ in range(L + 1)]
                    # hold the stream ~4 ms so the host enqueues every launch
                    # first: the events then time the GPU, not Python + ctypes
                    torch.cuda._sleep(8_000_000)
                    ev[0].record(stream)
                    for layer in range(L):
                        launch(fn, layer)
                        ev[layer + 1].record(stream)
                    torch.cuda.synchronize()
                    times += [ev[i].elapsed_time(ev[i + 1]) for i in range(L)]
                    span = ev[0].elapsed_time(ev[L])
                # the same L launches with no event between them (one pair around all)
                torch.cuda._sleep(8_000_000)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                for layer in range(L):
                    launch(fn, layer)
                e1.record(stream)
                torch.cuda.synchronize()
                per_launch_noev = e0.elapsed_time(e1) / L
            med = statistics.median(times)
            gbs = 2 * payload / (med / 1e3) / 1e9
            variant = "unit-affine" if args.affine else os.environ.get("TKV_PAGED_KERNEL", "unit")
            print(json.dumps({"kernel": name, "variant": variant, "bpt": bpt, "launch_mib": round(payload / 2**20, 2),
                              "launch_ms_median": round(med, 5), "launch_ms_min": round(min(times), 5),
                              "gbs": round(gbs, 1), "frac": round(gbs / peak, 4),
                              "back_to_back_gbs": round(2 * payload * L / (span / 1e3) / 1e9, 1),
                              "no_events_ms_per_launch": round(per_launch_noev, 5),
                              "no_events_gbs": round(2 * payload / (per_launch_noev / 1e3) / 1e9, 1),
                              "no_events_frac": round(2 * payload / (per_launch_noev / 1e3) / 1e9 / peak, 4),
                              "peak": peak}), flush=True)
        variant = os.environ.get("TKV_PAGED_KERNEL", "unit")
        for name, fn in (("K1 gather", lib_.tkv_gather_layers), ("K2 scatter", lib_.tkv_scatter_layers)):
            # one launch over all layers (bench.py's value loop shape) ...
            t = timed(lambda: check(fn(ct.byref(layout), d_desc.data_ptr(), d_tb_all.data_ptr(), len(descs),
                                       int(tb_all[-1]), 0, L, ppt_all, ao, args.ctas, stream.cuda_stream)), reps=5)
            print(json.dumps({"kernel": name + " all layers", "variant": variant, "bpt": bpt,
                              "launch_mib": round(L * payload / 2**20, 1), "launch_ms_median": round(t, 4),
                              "gbs": round(2 * L * payload / (t / 1e3) / 1e9, 1),
                              "frac": round(2 * L * payload / (t / 1e3) / 1e9 / peak, 4)}), flush=True)
            # ... and one page: the fixed per-launch cost
            t = timed(lambda: check(fn(ct.byref(layout), d_desc.data_ptr(), d_tb_one.data_ptr(), 1, 1, 0, 1, ppt,
                                       ao, args.ctas, stream.cuda_stream)))
            print(json.dumps({"kernel": name + " one page (launch floor)", "variant": variant, "bpt": bpt,
                              "launch_kib": 16 * bpt / 1024, "launch_ms_median": round(t, 5)}), flush=True)
        # a plain contiguous device copy of the same bytes (torch copy_), on
        # distinct ring regions per launch so neither side is in L2
        with torch.cuda.stream(stream):
            views = [(ring[(2 * i) * payload:(2 * i + 1) * payload], ring[(2 * i + 1) * payload:(2 * i + 2) * payload])
                     for i in range(min(20, L // 2))]
            for a, b in views[:3]:
                b.copy_(a)
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(len(views) + 1)]
            torch.cuda._sleep(8_000_000)
            ev[0].record(stream)
            for i, (a, b) in enumerate(views):
                b.copy_(a)
                ev[i + 1].record(stream)
            torch.cuda.synchronize()
            ce = statistics.median(ev[i].elapsed_time(ev[i + 1]) for i in range(len(views)))
            # and the smallest kernel torch can launch: the per-launch floor of this timing method
            tiny = torch.zeros(1, device=dev)
            tiny.add_(1)
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(21)]
            torch.cuda._sleep(8_000_000)
            ev[0].record(stream)
            for i in range(20):
                tiny.add_(1)
                ev[i + 1].record(stream)
            torch.cuda.synchronize()
            floor = statistics.median(ev[i].elapsed_time(ev[i + 1]) for i in range(20))
        print(json.dumps({"kernel": "torch copy_ (D2D, same bytes, not L2-resident)", "bpt": bpt,
                          "launch_ms_median": round(ce, 5), "gbs": round(2 * payload / (ce / 1e3) / 1e9, 1),
                          "frac": round(2 * payload / (ce / 1e3) / 1e9 / peak, 4),
                          "tiny_kernel_ms": round(floor, 5)}), flush=True)
        e.release_query(q)
        e.close()
        del ring
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
