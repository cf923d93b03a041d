"""Host<->device bandwidth and streamed-apply chunking on one GPU:
  python tools/stream_probe.py"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_04644_b200 as sk  # noqa: E402
from paper_2604_04644_b200 import operators as ops  # noqa: E402

n = 294 << 20
h = torch.empty(n // 8, dtype=torch.float64, pin_memory=True)
h2 = torch.empty(n // 8, dtype=torch.float64, pin_memory=True)
d = torch.empty(n // 8, dtype=torch.float64, device="cuda")
d2 = torch.empty(n // 8, dtype=torch.float64, device="cuda")
res = {}
for name, fn in (("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(d, non_blocking=True))):
    fn(); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    res[name + "_gbs"] = 5 * n / (time.perf_counter() - t) / 1e9
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(5):
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize()
res["duplex_gbs_each"] = 5 * n / (time.perf_counter() - t) / 1e9
E = 1 << 20
b = sk.build_shape_basis(sk.Shape.TET, 4)
fac = sk.make_synthetic_factors(b, sk.GeometryClass.DEFORMED, E, seed=0)
blk = sk.Block(b, fac, sk.FieldState.COEFF, 1, 1)
blk.set_elements(np.random.default_rng(0).uniform(-1, 1, (1, b.n_modes, E)))
out = blk.like(sk.FieldState.COEFF)
blk.payload(0)
for chunks in (8, 16, 32, 64):
    ops.STREAM_CHUNK_ELEMENTS = E // chunks
    ts = []
    for it in range(6):
        blk.host(sk.AccessQualifier.READ_WRITE)
        torch.cuda.synchronize()
        t = time.perf_counter()
        sk.helmholtz_apply(blk, 1.0, out=out)
        out.host()
        ts.append(time.perf_counter() - t)
    res[f"e2e_gdofs_chunks{chunks}"] = b.n_modes * E / min(ts[1:]) / 1e9
print(json.dumps(res))
