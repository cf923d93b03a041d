"""Benchmark: Helmholtz apply throughput (GDOF/s) on B200, BASELINE config 2.

Workload (BASELINE.json configs[1]): Helmholtz operator (collocated, lam=1)
on a synthetic deformed tetrahedral mesh, P=4, 2^20 elements per GPU, FP64,
inputs resident in HBM (8.96 GB of geometry per apply >> 126 MB L2, so no
flush is needed between steps).  One process per GPU; every rank owns a
contiguous element range of the same seeded mesh (weak scaling, no
collective in the timed region); time = max over ranks of CUDA-event time.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl sk|reference]

``--impl reference`` times the reference algorithm on the host cores (the
numpy oracle restatement of speckern's sum-factorised operators; the
reference is pure Python, so there is no compiled reference to time).
"""

from __future__ import annotations

import os

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("OMP_NUM_THREADS", "1")

import argparse  # noqa: E402
import json  # noqa: E402
import statistics  # noqa: E402
import subprocess  # noqa: E402
import sys  # noqa: E402
import time  # noqa: E402

import numpy as np  # noqa: E402

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SHAPE, ORDER, E_PER_GPU, LAM, SEED = "tet", 4, 1 << 20, 1.0, 0
METRIC = "Helmholtz apply GDOF/s (tet, P=4, deformed, FP64)"
UNIT = "GDOF/s"


WORKLOADS = {
    # BASELINE configs[1]: Helmholtz, tet, P=4, ~10^6 deformed elements per GPU
    "tet4": {"blocks": [("tet", 4, 1 << 20)],
             "metric": METRIC,
             "name": "helmholtz_coll tet P=4 deformed, 2^20 elements per GPU (BASELINE configs[1])"},
    # BASELINE configs[3]: mixed hex/prism/pyr/tet Helmholtz, P=6, sharded
    "mixed6": {"blocks": [("hex", 6, 1 << 17), ("prism", 6, 1 << 17), ("pyr", 6, 1 << 17), ("tet", 6, 1 << 17)],
               "metric": "Helmholtz apply GDOF/s (mixed hex/prism/pyr/tet, P=6, deformed, FP64)",
               "name": "helmholtz_coll mixed hex/prism/pyr/tet P=6 deformed, 2^17 elements per shape per GPU "
                       "(BASELINE configs[3])"},
    # BASELINE configs[4]: assembled C0 variant (hex, P=4), z-slab per GPU,
    # NCCL exchange of the shared DOF layers inside the timed region
    "c0hex": {"blocks": [("hex", 4, 64 * 64 * 64)],
              "metric": "Assembled C0 Helmholtz apply GDOF/s (global DOFs, hex P=4, deformed, FP64)",
              "name": "assembled C0 helmholtz hex P=4, 64x64x64 elements per GPU (z-slabs), "
                      "NCCL neighbour exchange of shared DOF layers (BASELINE configs[4])"},
}


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0}, "fallback"


def _config(wl, spec, ws):
    step_bytes = 0
    for shape, P, e in spec:
        from oracle.elements import mode_count, qcounts

        q = qcounts(shape, P)
        step_bytes += 8 * (2 * mode_count(shape, P) + 7 * q[0] * q[1] * q[2]) * e
    return {
        "workload": wl["name"],
        "blocks": [{"shape": s, "order": P, "elements_per_gpu": e} for s, P, e in spec],
        "elements_total": sum(e for _, _, e in spec) * ws,
        "lam": LAM,
        "geometry": "deformed (seeded sinusoidal, reference geometry.py:275-300)",
        "l2": f"inputs > L2 ({step_bytes / 1e9:.2f} GB per step per GPU), no flush",
        "parallelism": f"elements sharded contiguously over {ws} GPU(s), no collective",
    }


class Clocks:
    """nvidia-smi sampler running during the timed region."""

    Q = (
        "clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
        "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap"
    )

    def __init__(self, dev: int):
        self.dev = dev
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits", "-i", str(self.dev), "-lms", "50"],
                stdout=subprocess.PIPE,
                stderr=subprocess.DEVNULL,
                text=True,
            )
        except OSError:
            self.p = None
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.p is not None:
            self.p.terminate()
            try:
                out, _ = self.p.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.p.kill()
                out, _ = self.p.communicate()
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            try:
                sm.append(float(f[0]))
                mx = max(mx, float(f[1]))
            except (ValueError, IndexError):
                continue
            for name, v in zip(names, f[2:]):
                if v.lower() == "active":
                    reasons.add(name)
        return {
            "sm_mhz": statistics.median(sm) if sm else None,
            "sm_max_mhz": mx or None,
            "reasons": sorted(reasons),
            "samples": len(sm),
        }


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


_CPU_STATE: dict = {}


def _cpu_init(counter, per_core, blocks):
    """Worker initialiser: claim a distinct contiguous slice of one block of
    the workload (blocks round-robin over workers) and build it with the
    oracle (geometry, coefficients, lam payload)."""
    import oracle as O
    from oracle.geom import deformed_coords, payload_lam

    with counter.get_lock():
        idx = counter.value
        counter.value += 1
    k = idx % len(blocks)
    shape, P = blocks[k]
    first, n = (idx // len(blocks)) * per_core, per_core
    el = O.element(shape, P)
    geo = O.deformed_geometry_from_coords(el, deformed_coords(el, O.deformation_params(n, SEED + k, first=first)))
    x = np.random.default_rng([SEED, O.SHAPE_INDEX[shape], P, 1, first]).uniform(-1.0, 1.0, (n, el.nm)).T
    # the lam payload is cached per block in the reference (field_block.py:309-321)
    _CPU_STATE["slice"] = (el, geo, np.ascontiguousarray(x), payload_lam(el, geo))


def _cpu_task(reps):
    """Apply the reference Helmholtz to this worker's slice ``reps`` times."""
    import oracle as O

    el, geo, x, lp = _CPU_STATE["slice"]
    for _ in range(reps):
        O.helmholtz_coll(el, geo, x, LAM, lam_payload=lp)
    return el.nm * x.shape[1] * reps


class CpuReference:
    """The reference algorithm (numpy oracle restatement of speckern's
    sum-factorised Helmholtz, operators.py:670-699) on the host cores: one
    worker process per core, each on its own contiguous element slice of the
    workload (numpy is GIL-bound at these matrix sizes, so threads do not
    scale).  Throughput = DOF / parent wall time of one pass over all slices."""

    def __init__(self, cores: int, per_core: int = 4096, blocks=((SHAPE, ORDER),)):
        import multiprocessing as mp

        ctx = mp.get_context("spawn")
        self.cores, self.per_core = cores, per_core
        self.pool = ctx.Pool(cores, initializer=_cpu_init, initargs=(ctx.Value("i", 0), per_core, tuple(blocks)))
        self.reps = 1
        self.run(1)  # warm up every worker

    def run(self, reps: int):
        t0 = time.perf_counter()
        dof = sum(self.pool.map(_cpu_task, [reps] * self.cores, chunksize=1))
        return dof, time.perf_counter() - t0

    def calibrate(self, seconds: float) -> int:
        dof, dt = self.run(1)
        self.reps = max(1, int(round(seconds / max(dt, 1e-6))))
        return self.reps

    def close(self):
        self.pool.close()
        self.pool.join()


def run_reference(args, ws, rank):
    if rank != 0:
        return
    wl = WORKLOADS[args.workload]
    spec = [(s, P, args.elements or e) for s, P, e in wl["blocks"]]
    cores = os.cpu_count() or 1
    per_core = int(os.environ.get("SK_BENCH_CPU_PER_CORE", "4096"))
    if any(P >= 6 for _, P, _ in spec):
        per_core = max(1, per_core // 8)
    ref = CpuReference(cores, per_core, [(s, P) for s, P, _ in spec])
    step_s = max(0.3, min(3.0, 150.0 / max(1, args.steps + args.warmup)))
    reps = ref.calibrate(step_s)
    for _ in range(args.warmup):
        ref.run(reps)
    vals = []
    for _ in range(args.steps):
        dof, dt = ref.run(reps)
        vals.append(dof / dt / 1e9)
    ref.close()
    value = statistics.median(vals)
    n_sample = ref.per_core * cores
    line = {
        "impl": "reference",
        "metric": wl["metric"],
        "value": value,
        "unit": UNIT,
        "n_gpus": ws,
        "steps": args.steps,
        "warmup": args.warmup,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (seeded reference mesh)",
        "config": _config(wl, spec, ws),
        "cpu_baseline": {
            "value": value,
            "unit": UNIT,
            "cores": cores,
            "kind": "port",
            "sample": f"{n_sample} elements ({ref.per_core} per core process) x {reps} passes per step, median of {args.steps} steps",
        },
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_device(args, ws, rank, local):
    import torch

    import paper_2604_04644_b200 as sk
    from paper_2604_04644_b200 import _lib
    import oracle as O

    torch.cuda.set_device(local)
    dist = None
    if ws > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.cuda.current_device()
    wl = WORKLOADS[args.workload]
    spec = [(s, P, args.elements or e) for s, P, e in wl["blocks"]]
    if args.workload == "c0hex":
        return run_c0(args, ws, rank, dist, dev, wl)

    # every rank owns a contiguous slice of each block of the seeded mesh
    # (weak scaling: elements per GPU fixed); block k uses seed SEED + k
    blocks, outs = [], []
    for k, (shape, P, E) in enumerate(spec):
        basis = sk.build_shape_basis(sk.Shape(shape), P)
        fac = sk.make_synthetic_factors(basis, sk.GeometryClass.DEFORMED, E, seed=SEED + k, first=rank * E)
        blk = sk.Block(basis, fac, sk.FieldState.COEFF, 1, 1)
        key = [SEED, O.SHAPE_INDEX[shape], P, 1] + ([rank] if rank else [])
        x = np.random.default_rng(key).uniform(-1.0, 1.0, size=(E, basis.n_modes)).T
        blk.set_elements(x[None])
        blk.payload(_lib.SK_PAYLOAD_HELMHOLTZ)  # one-time geometry payload (untimed, as Block.payload)
        blocks.append(blk)
        outs.append(blk.like(sk.FieldState.COEFF))
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    nb = len(blocks)
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(nb + 1)] for _ in range(args.steps)]

    def step(marks=None):
        for b, (blk, out) in enumerate(zip(blocks, outs)):
            if marks is not None:
                marks[b].record(stream)
            sk.helmholtz_apply(blk, LAM, out=out)
        if marks is not None:
            marks[nb].record(stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n0 = _lib.launch_count()
    with Clocks(dev) as clk:
        torch.cuda.synchronize()
        t0.record(stream)
        for i in range(args.steps):
            step(ev[i])
        t1.record(stream)
        torch.cuda.synchronize()
    launches = _lib.launch_count() - n0
    if dist:
        dist.barrier()
    ms = t0.elapsed_time(t1)
    per_block_ms = [sum(ev[i][b].elapsed_time(ev[i][b + 1]) for i in range(args.steps)) / args.steps for b in range(nb)]
    tmax = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if dist:
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
    ms_max = float(tmax.item())
    ndof_rank = sum(b.basis.n_modes * b.n_elements for b in blocks)
    ndof = ndof_rank * ws
    value = ndof * args.steps / (ms_max / 1e3) / 1e9

    # e2e through the public API with host buffers: H2D of the step's
    # coefficients (pinned), apply, D2H of the result, every step
    e2e_steps = max(3, min(args.steps, 10))
    h2d = d2h = sum(8 * b.basis.n_modes * b.padded_elements for b in blocks)
    for _ in range(2):
        for blk, out in zip(blocks, outs):
            blk.host(sk.AccessQualifier.READ_WRITE)
            sk.helmholtz_apply(blk, LAM, out=out).host()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    w0 = time.perf_counter()
    for _ in range(e2e_steps):
        for blk, out in zip(blocks, outs):
            blk.host(sk.AccessQualifier.READ_WRITE)  # host copy is now the live one
            sk.helmholtz_apply(blk, LAM, out=out)  # -> H2D transfer + kernel
            out.host()  # -> D2H transfer of the result
    torch.cuda.synchronize()
    we = torch.tensor([time.perf_counter() - w0], dtype=torch.float64, device="cuda")
    if dist:
        dist.all_reduce(we, op=dist.ReduceOp.MAX)
    e2e_val = ndof * e2e_steps / float(we.item()) / 1e9

    # roofline of the dominant kernel: algorithmic bytes per launch / its
    # average duration (CUDA events on the launching stream)
    peaks, src = _peaks()
    dom = int(np.argmax(per_block_ms))
    db = blocks[dom]
    bytes_per_launch = sk.operator_bytes(sk.OperatorKind.HELMHOLTZ_COLL, db.shape, db.basis.order, True, LAM) * db.n_elements
    achieved = bytes_per_launch / (per_block_ms[dom] / 1e3) / 1e9
    step_bytes = sum(sk.operator_bytes(sk.OperatorKind.HELMHOLTZ_COLL, b.shape, b.basis.order, True, LAM) * b.n_elements
                     for b in blocks)
    traffic = None
    prof = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(prof):
        try:
            with open(prof) as fh:
                per_el = json.load(fh).get(f"{db.shape.value}_P{db.basis.order}_helm_per_element_bytes")
            traffic = per_el * db.n_elements if per_el else None
        except (OSError, ValueError):
            traffic = None

    if rank == 0:
        cores = os.cpu_count() or 1
        ref = CpuReference(cores, 4096 if max(P for _, P, _ in spec) < 6 else 512, [(s, P) for s, P, _ in spec])
        reps = ref.calibrate(10.0)
        dofs, dt = ref.run(reps)
        ref.close()
        cpu_v = dofs / dt / 1e9
        cfg = _config(wl, spec, ws)
        line = {
            "metric": wl["metric"],
            "value": value,
            "unit": UNIT,
            "n_gpus": ws,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms_max / args.steps,
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic (seeded reference mesh, device geometry builder)",
            "config": cfg,
            "roofline": {
                "bound": "hbm",
                "achieved": achieved,
                "peak": peaks.get("hbm_gbs", 6650.0),
                "unit": "GB/s",
                "frac": achieved / peaks.get("hbm_gbs", 6650.0),
                "traffic": traffic,
                "peak_source": src,
                "bytes_per_launch": bytes_per_launch,
                "kernel": f"helmholtz {db.shape.value} P={db.basis.order}",
                "step_frac": step_bytes / (ms / 1e3 / args.steps) / 1e9 / peaks.get("hbm_gbs", 6650.0),
            },
            "cpu_baseline": {
                "value": cpu_v,
                "unit": UNIT,
                "cores": cores,
                "kind": "port",
                "sample": f"{ref.per_core * cores} elements of the workload ({cores} processes x {ref.per_core}, "
                          f"blocks round-robin) x {reps} passes: {dofs / 1e6:.0f} MDOF in {dt:.1f} s",
            },
            "e2e": {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
            "gpu_launches": launches,
            "clocks": clk.summary(),
        }
        if nb > 1:
            line["per_block_ms"] = {f"{b.shape.value}": m for b, m in zip(blocks, per_block_ms)}
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def run_c0(args, ws, rank, dist, dev, wl):
    """Assembled C0 Helmholtz: gather -> elemental kernel -> scatter -> NCCL
    exchange of the two shared DOF layers, all inside the timed region."""
    import torch

    from paper_2604_04644_b200 import _lib
    from paper_2604_04644_b200.assembly import C0HexMesh

    n = 64 if not args.elements else max(1, round(args.elements ** (1.0 / 3.0)))
    P = 4
    mesh = C0HexMesh(n, n, n * ws, P, rank=rank, world=ws)
    x = torch.empty(mesh.n_dofs, dtype=torch.float64, device="cuda").uniform_(-1.0, 1.0)
    mesh.block.payload(_lib.SK_PAYLOAD_HELMHOLTZ)
    for _ in range(args.warmup):
        mesh.helmholtz(x, LAM)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    stream = torch.cuda.current_stream()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n0 = _lib.launch_count()
    with Clocks(dev) as clk:
        torch.cuda.synchronize()
        t0.record(stream)
        for _ in range(args.steps):
            mesh.helmholtz(x, LAM)
        t1.record(stream)
        torch.cuda.synchronize()
    launches = _lib.launch_count() - n0
    ms = t0.elapsed_time(t1)
    tmax = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if dist:
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
    ms_max = float(tmax.item())
    n_global = (n * P + 1) ** 2 * (n * ws * P + 1)
    value = n_global * args.steps / (ms_max / 1e3) / 1e9
    # e2e: host DOF vector in, host result out, every step
    xh = torch.empty(mesh.n_dofs, dtype=torch.float64).pin_memory().uniform_(-1.0, 1.0)
    yh = torch.empty_like(xh).pin_memory()
    e2e_steps = max(3, min(args.steps, 10))
    torch.cuda.synchronize()
    w0 = time.perf_counter()
    for _ in range(e2e_steps):
        yh.copy_(mesh.helmholtz(xh.to("cuda", non_blocking=True), LAM))
    torch.cuda.synchronize()
    we = torch.tensor([time.perf_counter() - w0], dtype=torch.float64, device="cuda")
    if dist:
        dist.all_reduce(we, op=dist.ReduceOp.MAX)
    e2e_val = n_global * e2e_steps / float(we.item()) / 1e9
    peaks, src = _peaks()
    import paper_2604_04644_b200 as sk

    bel = sk.operator_bytes(sk.OperatorKind.HELMHOLTZ_COLL, sk.Shape.HEX, P, True, LAM)
    step_bytes = bel * mesh.E + 2 * 8 * mesh.n_dofs
    achieved = step_bytes / (ms / 1e3 / args.steps) / 1e9
    if rank == 0:
        line = {
            "metric": wl["metric"],
            "value": value,
            "unit": UNIT,
            "n_gpus": ws,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms_max / args.steps,
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic (conforming deformed hex mesh, device geometry builder)",
            "config": {"workload": wl["name"], "elements_per_gpu": mesh.E, "global_dofs": n_global, "order": P,
                       "lam": LAM, "l2": f"inputs > L2 ({step_bytes / 1e9:.2f} GB per step per GPU), no flush",
                       "parallelism": f"z-slabs over {ws} GPU(s), NCCL P2P exchange of 2 DOF layers per step"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peaks.get("hbm_gbs", 6650.0), "unit": "GB/s",
                         "frac": achieved / peaks.get("hbm_gbs", 6650.0), "traffic": None, "peak_source": src,
                         "bytes_per_launch": step_bytes, "kernel": "whole step (gather + helmholtz + scatter)"},
            "cpu_baseline": None,
            "e2e": {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": 8 * mesh.n_dofs,
                    "d2h_bytes_per_step": 8 * mesh.n_dofs},
            "gpu_launches": launches,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def run_reference_sweep(args):
    """Reference CPU path (oracle port of speckern's sum-factorised Helmholtz,
    all host cores) per shape x order: one JSON line each, to sit beside the
    device sweep (tools/sweep.py).  Bounded samples (~2 s per case)."""
    cores = os.cpu_count() or 1
    for shape in ("hex", "prism", "pyr", "tet"):
        for P in range(1, 11):
            per_core = max(8, int(2048 * (5.0 / (P + 1)) ** 3))
            ref = CpuReference(cores, per_core, [(shape, P)])
            reps = ref.calibrate(1.5)
            vals = []
            for _ in range(3):
                dof, dt = ref.run(reps)
                vals.append(dof / dt / 1e9)
            ref.close()
            print(json.dumps({"impl": "reference", "op": "helm", "shape": shape, "P": P,
                              "gdof_s": statistics.median(vals), "cores": cores, "kind": "port",
                              "sample": f"{per_core * cores} elements x {reps} passes, median of 3"}), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["sk", "reference"], default="sk")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="tet4")
    ap.add_argument("--elements", type=int, default=0, help="override elements per block per GPU")
    ap.add_argument("--sweep", action="store_true", help="with --impl reference: CPU GDOF/s per shape x order")
    args = ap.parse_args()
    ws, rank, local = _dist()
    if args.impl == "reference" and args.sweep:
        if rank == 0:
            run_reference_sweep(args)
        return
    if args.impl == "reference":
        run_reference(args, ws, rank)
        return
    run_device(args, ws, rank, local)


if __name__ == "__main__":
    main()
