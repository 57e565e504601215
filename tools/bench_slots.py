"""K1/K2 with a vLLM-style per-token slot_mapping (page_tokens = 1 layout,
K and V planes per layer, scattered slots): HBM GB/s of the algorithmic
bytes (2 x payload) for 16K tokens x 80 layers x 4096 B (5 GiB per launch),
the same payload as the bench's block-table launches."""
import ctypes as ct
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2510_09665_b200._lib import check, lib  # noqa: E402
from paper_2510_09665_b200.api import PagedLayoutC, XferDescC, plan_tiles  # noqa: E402


def main(L=80, n_tok=16384, hd=2048, reps=5):
    rng = np.random.default_rng(1)
    n_slots = n_tok + 1024
    kv = [torch.empty(2 * n_slots * hd, dtype=torch.uint8, device="cuda") for _ in range(L)]
    bases = torch.tensor([t.data_ptr() for t in kv], dtype=torch.int64).cuda()
    res = {}
    for kind in ("block-ordered", "random"):
        slots = (np.arange(n_tok) if kind == "block-ordered" else rng.permutation(n_slots)[:n_tok]).astype(np.int32)
        tab = torch.from_numpy(slots).cuda()
        ch = torch.empty(L * n_tok * 2 * hd, dtype=torch.uint8, device="cuda")
        d = XferDescC(chunk=ch.data_ptr(), layer_stride=n_tok * 2 * hd, table_dev=tab.data_ptr(),
                      table_stride=n_tok, first_page=0, n_tokens=n_tok)
        tb, ppt = plan_tiles([d], 1, hd, L)
        dd = torch.frombuffer(bytearray(bytes(d)), dtype=torch.uint8).cuda()
        dt = torch.from_numpy(tb.view(np.int32)).cuda()
        lay = PagedLayoutC(base=0, layer_base_dev=bases.data_ptr(), page_stride=hd, plane_stride=n_slots * hd,
                           token_stride=hd, plane_bytes=hd, n_planes=2, page_tokens=1, bpt=2 * hd, shared_table=1)
        for name, fn in (("gather", lib().tkv_gather_layers), ("scatter", lib().tkv_scatter_layers)):
            def go():
                check(fn(ct.byref(lay), dd.data_ptr(), dt.data_ptr(), 1, int(tb[-1]), 0, L, ppt,
                         d.chunk | d.layer_stride, 0, None))
            go()
            torch.cuda.synchronize()
            ts = []
            for _ in range(reps):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                go()
                b.record()
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b))
            res[f"{kind} {name}"] = round(2 * L * n_tok * 2 * hd / min(ts) / 1e6, 1)
        del ch
    print(json.dumps({"slot_mapping_k1k2_hbm_gbps": res, "payload_bytes": L * n_tok * 2 * hd,
                      "layout": "vLLM K/V planes per layer, page_tokens = 1 (table = slot_mapping)"}))


if __name__ == "__main__":
    main()
