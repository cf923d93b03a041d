"""PCIe pipeline probe: the streamed apply's copy pattern without the
kernel (H2D chunk i on one stream; D2H chunk i on another after it), with
the mass kernel, and with the Helmholtz kernel, to split the e2e step time.
GPU box: python tools/pcie_pipeline.py"""

import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

n = 293601280 // 8
hin = torch.empty(n, dtype=torch.float64, pin_memory=True)
hout = torch.empty(n, dtype=torch.float64, pin_memory=True)
din = torch.empty(n, dtype=torch.float64, device="cuda")
dout = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def pipeline(nch, work=None):
    bounds = [i * n // nch for i in range(nch + 1)]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    evs = []
    for i in range(nch):
        a, b = bounds[i], bounds[i + 1]
        with torch.cuda.stream(s1):
            din[a:b].copy_(hin[a:b], non_blocking=True)
            e = torch.cuda.Event()
            e.record()
        with torch.cuda.stream(s2):
            s2.wait_event(e)
            if work is not None:
                work(a, b)
            hout[a:b].copy_(dout[a:b], non_blocking=True)
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) * 1e3


def axpy(a, b):  # an HBM-streaming kernel on the chunk (reads din, writes dout)
    torch.mul(din[a:b], 1.0001, out=dout[a:b])


for nch in (1, 8, 16, 32):
    for name, w in (("copies", None), ("copies+axpy", axpy)):
        best = min(pipeline(nch, w) for _ in range(4))
        print(json.dumps({"chunks": nch, "mode": name, "ms": round(best, 3),
                          "gbs_per_dir": round(8 * n / best / 1e6, 1)}), flush=True)
