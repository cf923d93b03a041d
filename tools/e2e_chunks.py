"""e2e (host buffers in and out, every step) of the bench's headline
workload vs the streamed chunk count.  GPU box:
  python tools/e2e_chunks.py > gpurun_out/e2e_chunks.jsonl"""

import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2604_04644_b200 as sk  # noqa: E402
from paper_2604_04644_b200 import operators as ops  # noqa: E402

E = 1 << 20
b = sk.build_shape_basis(sk.Shape.TET, 4)
fac = sk.make_synthetic_factors(b, sk.GeometryClass.DEFORMED, E, seed=0)
blk = sk.Block(b, fac, sk.FieldState.COEFF, 1, 1)
blk.device(sk.AccessQualifier.WRITE_ONLY).uniform_(-1, 1)
out = blk.like(sk.FieldState.COEFF)
sk.helmholtz_apply(blk, 1.0, out=out)
torch.cuda.synchronize()
ndof = b.n_modes * E
for nch, direct in ((0, True), (0, False), (-1, True), (8, True), (16, True), (32, True)):
    # 0: default ramped schedule; -1: default with the ramp off (SK_STREAM_RAMP=0);
    # direct: kernels store straight into the pinned host output (no D2H stage)
    os.environ["SK_STREAM_RAMP"] = "0" if nch == -1 else "1"
    ops.STREAM_CHUNK_ELEMENTS = -(-E // nch) if nch > 0 else 0
    ops.STREAM_DIRECT_OUT = direct
    for _ in range(2):
        blk.host(sk.AccessQualifier.READ_WRITE)
        sk.helmholtz_apply(blk, 1.0, out=out).host()
    torch.cuda.synchronize()
    best = 1e9
    for rep in range(3):
        t0 = time.perf_counter()
        for _ in range(8):
            blk.host(sk.AccessQualifier.READ_WRITE)
            sk.helmholtz_apply(blk, 1.0, out=out)
            out.host()
        torch.cuda.synchronize()
        best = min(best, (time.perf_counter() - t0) / 8)
    print(json.dumps({"chunks": nch, "direct_out": direct, "ms_per_step": best * 1e3, "e2e_gdof_s": ndof / best / 1e9}),
          flush=True)

# where the step time goes (default schedule): host time inside the apply
# call, device time of the apply (events on the current stream), wall
ops.STREAM_CHUNK_ELEMENTS = 0
ops.STREAM_DIRECT_OUT = True
os.environ["SK_STREAM_RAMP"] = "1"
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for _ in range(3):
    blk.host(sk.AccessQualifier.READ_WRITE)
    torch.cuda.synchronize()
    w0 = time.perf_counter()
    ev0.record()
    h0 = time.perf_counter()
    sk.helmholtz_apply(blk, 1.0, out=out)
    h1 = time.perf_counter()
    ev1.record()
    out.host()
    w1 = time.perf_counter()
    torch.cuda.synchronize()
    print(json.dumps({"wall_ms": (w1 - w0) * 1e3, "host_call_ms": (h1 - h0) * 1e3,
                      "device_ms": ev0.elapsed_time(ev1)}), flush=True)
