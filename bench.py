"""Benchmark: Helmholtz apply throughput (GDOF/s) on B200.

Default workload (BASELINE.json configs[1]): Helmholtz operator (collocated,
lam=1) on a synthetic deformed tetrahedral mesh, P=4, 2^20 elements per GPU,
FP64, inputs resident in HBM (9.4 GB of traffic per apply >> 126 MB L2, so
no flush is needed between steps).  One process per GPU; every rank owns a
contiguous element range of the same seeded mesh (weak scaling, no
collective in the timed region); time = max over ranks of CUDA-event time.

The same JSON line carries ``per_shape_P`` -- the BASELINE metric itself
("Helmholtz apply GDOF/s per shape vs P; % of roofline"): every shape at
P=2..10 (deformed, plus regular, plus the recomputed-metric variant), and
mass / stiffness on every shape at P=2..8 (configs[2] names prism and pyr); each cell >= 1 GB of algorithmic traffic per apply,
with its roofline fraction, a sampled-element parity error against the CPU
oracle and the SM clocks sampled while it ran.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl sk|reference]
                  [--workload tet4|hex4|mixed6|c0hex] [--sweep auto|on|off]

``--gpus N`` (N > 1) without a torchrun environment re-launches itself under
``torch.distributed.run`` with N ranks on 127.0.0.1.

``--impl reference`` times the reference's own CPU implementation on the
host cores: the unmodified ``speckern`` package installed in
``baseline/_ref`` (``apply_operator(HELMHOLTZ_COLL, block, SUM_FAC, lam)``,
one worker process per core), or -- when it is not installed -- the numpy
oracle restatement of the same algorithm.
"""

from __future__ import annotations

import os

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("OMP_NUM_THREADS", "1")

import argparse  # noqa: E402
import json  # noqa: E402
import socket  # noqa: E402
import statistics  # noqa: E402
import subprocess  # noqa: E402
import sys  # noqa: E402
import threading  # noqa: E402
import time  # noqa: E402

import numpy as np  # noqa: E402

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
REF_DIR = os.path.join(ROOT, "baseline", "_ref")

SHAPE, ORDER, E_PER_GPU, LAM, SEED = "tet", 4, 1 << 20, 1.0, 0
METRIC = "Helmholtz apply GDOF/s (tet, P=4, deformed, FP64)"
UNIT = "GDOF/s"
SHAPES = ("hex", "prism", "pyr", "tet")

WORKLOADS = {
    # BASELINE configs[1]: Helmholtz, tet, P=4, ~10^6 deformed elements per GPU
    "tet4": {"blocks": [("tet", 4, 1 << 20)],
             "metric": METRIC,
             "name": "helmholtz_coll tet P=4 deformed, 2^20 elements per GPU (BASELINE configs[1])"},
    # BASELINE configs[0]: Helmholtz, hex, P=4, 10^3 deformed elements (an
    # L2-resident latency figure: L2 flushed before every timed apply)
    "hex4": {"blocks": [("hex", 4, 1000)],
             "metric": "Helmholtz apply GDOF/s (hex, P=4, 10^3 deformed elements, cold L2, FP64)",
             "name": "helmholtz_coll hex P=4 deformed, 1000 elements per GPU (BASELINE configs[0])"},
    # BASELINE configs[4] "max elements per GPU": one apply streams ~115 GB
    # (payload + coefficients) of the 180 GB HBM
    "tet4max": {"blocks": [("tet", 4, 12_800_000)],
                "metric": "Helmholtz apply GDOF/s (tet, P=4, 12.8M deformed elements per GPU, FP64)",
                "name": "helmholtz_coll tet P=4 deformed, 12.8M elements per GPU (~115 GB resident, BASELINE configs[4])"},
    # BASELINE configs[3]: mixed hex/prism/pyr/tet Helmholtz, P=6, sharded
    "mixed6": {"blocks": [("hex", 6, 1 << 17), ("prism", 6, 1 << 17), ("pyr", 6, 1 << 17), ("tet", 6, 1 << 17)],
               "metric": "Helmholtz apply GDOF/s (mixed hex/prism/pyr/tet, P=6, deformed, FP64)",
               "name": "helmholtz_coll mixed hex/prism/pyr/tet P=6 deformed, 2^17 elements per shape per GPU "
                       "(BASELINE configs[3])"},
    # BASELINE configs[4]: assembled C0 variant (hex, P=4), z-slab per GPU,
    # NCCL exchange of the shared DOF layers inside the timed region
    # assembled C0 on an extruded triangulated prism mesh (signed maps)
    "c0prism": {"blocks": [("prism", 4, 2 * 48 * 48 * 48)],
                "metric": "Assembled C0 Helmholtz apply GDOF/s (global DOFs, prism P=4, deformed, FP64)",
                "name": "assembled C0 helmholtz prism P=4, 48x48 triangulated squares x 48 layers per GPU "
                        "(extrusion slabs), NCCL neighbour exchange of shared DOF layers (BASELINE configs[4])"},
    # assembled C0 on Kuhn-split cubes (tets in global vertex order)
    "c0tet": {"blocks": [("tet", 4, 6 * 40 * 40 * 40)],
              "metric": "Assembled C0 Helmholtz apply GDOF/s (global DOFs, tet P=4, deformed, FP64)",
              "name": "assembled C0 helmholtz tet P=4, 40^3 Kuhn-split cubes per GPU (z slabs), "
                      "NCCL neighbour exchange of shared DOF planes (BASELINE configs[4])"},
    # assembled C0 on six pyramids per cube (apex at the centre)
    "c0pyr": {"blocks": [("pyr", 4, 6 * 40 * 40 * 40)],
              "metric": "Assembled C0 Helmholtz apply GDOF/s (global DOFs, pyr P=4, deformed, FP64)",
              "name": "assembled C0 helmholtz pyr P=4, 40^3 cubes x 6 pyramids per GPU (z slabs), "
                      "NCCL neighbour exchange of shared DOF planes (BASELINE configs[4])"},
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


def _fp64_peak():
    """Measured FP64 peak on B200 (TFLOP/s): the higher of the DFMA-chain and
    DMMA microbenchmarks (profiles/fp64_peak.json, profiles/r01b/dmma_peak.json)."""
    vals = []
    try:
        with open(os.path.join(ROOT, "profiles", "fp64_peak.json")) as fh:
            vals.append(float(json.load(fh)["fp64_tflops"]))
    except (OSError, ValueError, KeyError):
        pass
    try:
        with open(os.path.join(ROOT, "profiles", "r01b", "dmma_peak.json")) as fh:
            vals.extend(float(v) for v in json.load(fh)["dmma_tflops"].values())
    except (OSError, ValueError, KeyError):
        pass
    return max(vals) if vals else 37.0


def _config(wl, spec, ws):
    step_bytes = 0
    for shape, P, e in spec:
        from oracle.elements import mode_count, qcounts

        q = qcounts(shape, P)
        step_bytes += 8 * (2 * mode_count(shape, P) + 7 * q[0] * q[1] * q[2]) * e
    l2 = (f"inputs > L2 ({step_bytes / 1e9:.2f} GB per step per GPU), no flush" if step_bytes > 4 * 126e6
          else f"inputs ({step_bytes / 1e6:.1f} MB) fit in L2: 256 MB L2 flush before every timed apply")
    return {
        "workload": wl["name"],
        "blocks": [{"shape": s, "order": P, "elements_per_gpu": e} for s, P, e in spec],
        "elements_total": sum(e for _, _, e in spec) * ws,
        "lam": LAM,
        "geometry": "deformed (seeded sinusoidal, reference geometry.py:275-300)",
        "l2": l2,
        "parallelism": f"elements sharded contiguously over {ws} GPU(s), no collective",
    }


# ---------------------------------------------------------------------------
# clocks: NVML sampled from a thread every ~5 ms for the whole run, so even a
# 30-ms timed region carries samples; summaries are taken per time window

_REASONS = {  # nvmlClocksEventReason* bits
    0x8: "hw_slowdown",
    0x40: "hw_thermal_slowdown",
    0x20: "sw_thermal_slowdown",
    0x4: "sw_power_cap",
    0x80: "hw_power_brake_slowdown",
}


class Clocks:
    """Background SM-clock / throttle-reason sampler (NVML; nvidia-smi when
    NVML is unavailable)."""

    def __init__(self, dev: int, period_s: float = 0.005):
        self.dev, self.period = dev, period_s
        self.samples: list = []  # (t, sm_mhz, reasons_mask)
        self.max_mhz = None
        self._stop = threading.Event()
        self._thr = None
        self._proc = None

    def start(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self._nvml_index())
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))

            def loop():
                while not self._stop.is_set():
                    try:
                        sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                        rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                        self.samples.append((time.perf_counter(), float(sm), int(rs)))
                    except Exception:  # noqa: BLE001 - sampling must never break the bench
                        pass
                    self._stop.wait(self.period)

            self._thr = threading.Thread(target=loop, daemon=True)
            self._thr.start()
        except Exception:  # noqa: BLE001
            self._start_smi()
        return self

    def _nvml_index(self) -> int:
        vis = os.environ.get("CUDA_VISIBLE_DEVICES")
        if vis:
            try:
                return int(vis.split(",")[self.dev])
            except (ValueError, IndexError):
                return self.dev
        return self.dev

    def _start_smi(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self._proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits", "-i", str(self._nvml_index()),
                 "-lms", "20"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self._proc = None

        def reader():
            names = [0x8, 0x40, 0x20, 0x4]
            for ln in self._proc.stdout:
                f = [x.strip() for x in ln.split(",")]
                try:
                    sm, mx = float(f[0]), float(f[1])
                except (ValueError, IndexError):
                    continue
                self.max_mhz = mx
                mask = 0
                for bit, v in zip(names, f[2:]):
                    if v.lower() == "active":
                        mask |= bit
                self.samples.append((time.perf_counter(), sm, mask))

        if self._proc is not None:
            self._thr = threading.Thread(target=reader, daemon=True)
            self._thr.start()

    def stop(self):
        self._stop.set()
        if self._proc is not None:
            self._proc.terminate()
        if self._thr is not None:
            self._thr.join(timeout=2)

    def summary(self, t0: float | None = None, t1: float | None = None, pad: float = 0.0):
        sel = [s for s in list(self.samples)
               if (t0 is None or s[0] >= t0 - pad) and (t1 is None or s[0] <= t1 + pad)]
        mask = 0
        for s in sel:
            mask |= s[2]
        return {
            "sm_mhz": statistics.median(s[1] for s in sel) if sel else None,
            "sm_min_mhz": min(s[1] for s in sel) if sel else None,
            "sm_max_mhz": self.max_mhz,
            "reasons": sorted(n for b, n in _REASONS.items() if mask & b),
            "samples": len(sel),
        }


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def _relaunch(args) -> int:
    """--gpus N > 1 outside torchrun: run this script under
    torch.distributed.run with N ranks (one per GPU) and return its status."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


# ---------------------------------------------------------------------------
# CPU reference (the reference arm and the cpu_baseline leg)

_CPU_STATE: dict = {}


def _ref_available() -> bool:
    return os.path.isdir(os.path.join(REF_DIR, "speckern"))


def _cpu_init(counter, per_core, blocks, kind):
    """Worker initialiser: build one block of the workload (blocks round-robin
    over workers).  kind "reference": the unmodified speckern from
    baseline/_ref (make_field + bench-style seeded coefficients,
    speckern/bench.py:167-172); kind "port": the oracle restatement on a
    distinct contiguous slice of the same seeded mesh."""
    with counter.get_lock():
        idx = counter.value
        counter.value += 1
    k = idx % len(blocks)
    shape, P = blocks[k]
    if kind == "reference":
        sys.path.insert(0, REF_DIR)
        from speckern.field_block import make_field
        from speckern.geometry import GeometryClass
        from speckern.operators import OperatorKind, Strategy
        from speckern.shapes import Shape

        fld = make_field(Shape[shape.upper()], P, GeometryClass.DEFORMED, per_core, seed=SEED + k)
        blk = fld.blocks[0]
        rng = np.random.default_rng([SEED, list(Shape).index(Shape[shape.upper()]), P, 1])
        blk.set_elements(np.ascontiguousarray(rng.uniform(-1.0, 1.0, (per_core, blk.n_data)).T)[None])
        _CPU_STATE["ref"] = (blk, OperatorKind.HELMHOLTZ_COLL, Strategy.SUM_FAC)
        return
    import oracle as O
    from oracle.geom import deformed_coords, payload_lam

    first, n = (idx // len(blocks)) * per_core, per_core
    el = O.element(shape, P)
    geo = O.deformed_geometry_from_coords(el, deformed_coords(el, O.deformation_params(n, SEED + k, first=first)))
    x = np.random.default_rng([SEED, O.SHAPE_INDEX[shape], P, 1, first]).uniform(-1.0, 1.0, (n, el.nm)).T
    # the lam payload is cached per block in the reference (field_block.py:309-321)
    _CPU_STATE["slice"] = (el, geo, np.ascontiguousarray(x), payload_lam(el, geo))


def _cpu_task(reps):
    """Apply the reference Helmholtz to this worker's block ``reps`` times."""
    if "ref" in _CPU_STATE:
        from speckern.operators import apply_operator

        blk, kind, strat = _CPU_STATE["ref"]
        for _ in range(reps):
            apply_operator(kind, blk, strat, LAM)
        return blk.basis.n_modes * blk.n_elements * reps
    import oracle as O

    el, geo, x, lp = _CPU_STATE["slice"]
    for _ in range(reps):
        O.helmholtz_coll(el, geo, x, LAM, lam_payload=lp)
    return el.nm * x.shape[1] * reps


class CpuReference:
    """The reference Helmholtz (speckern.operators.apply_operator
    HELMHOLTZ_COLL / SUM_FAC, operators.py:670-699, 724-746) on the host
    cores: one worker process per core, each applying it to its own block of
    the workload (numpy is GIL-bound at these matrix sizes, so threads do not
    scale).  Throughput = DOF / parent wall time of one pass over all
    workers."""

    def __init__(self, cores: int, per_core: int = 4096, blocks=((SHAPE, ORDER),), kind: str | None = None):
        import multiprocessing as mp

        ctx = mp.get_context("spawn")
        self.kind = kind or ("reference" if _ref_available() else "port")
        self.cores, self.per_core = cores, per_core
        self.pool = ctx.Pool(cores, initializer=_cpu_init,
                             initargs=(ctx.Value("i", 0), per_core, tuple(blocks), self.kind))
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


def _per_core(spec) -> int:
    per_core = int(os.environ.get("SK_BENCH_CPU_PER_CORE", "2048"))
    if any(P >= 6 for _, P, _ in spec):
        per_core = max(1, per_core // 8)
    return per_core


def run_reference(args, ws, rank):
    if rank != 0:
        return
    wl = WORKLOADS[args.workload]
    spec = [(s, P, args.elements or e) for s, P, e in wl["blocks"]]
    cores = os.cpu_count() or 1
    ref = CpuReference(cores, min(_per_core(spec), max(e for _, _, e in spec)), [(s, P) for s, P, _ in spec])
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
    what = ("unmodified speckern (baseline/_ref) apply_operator(HELMHOLTZ_COLL, SUM_FAC)" if ref.kind == "reference"
            else "oracle port of speckern's sum-factorised Helmholtz")
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
            "kind": ref.kind,
            "sample": f"{what}: {n_sample} elements ({ref.per_core} per core process) x {reps} passes per step, "
                      f"median of {args.steps} steps",
        },
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# per (shape, P) sweep: the BASELINE metric table

SWEEP_BYTES = 1.2e9  # algorithmic bytes per apply per cell (>= 1 GB, >> L2)
POOL = 1 << 16  # reference-seeded elements per pool, tiled to the cell size


def _cells(quick: bool, only=None):
    orders = (2, 4, 6, 8, 10) if quick else tuple(range(2, 11))
    if only:
        return [c for c in _cells(quick) if c[0] in only]
    out = []
    for s in SHAPES:
        for P in orders:
            out.append(("helm_deformed", "helm", True, s, P))
    for s in SHAPES:
        for P in orders:
            out.append(("helm_regular", "helm", False, s, P))
    for s in SHAPES:
        for P in orders:
            out.append(("helm_recompute", "helmp", True, s, P))
    for tab, op in (("mass_deformed", "mass"), ("stiff_deformed", "stiff")):
        for s in SHAPES:
            for P in (orders if quick else range(2, 9)):
                if P <= 8:
                    out.append((tab, op, True, s, P))
    return out


def _copy_ceiling(h2d: int, d2h: int, ndof: int) -> dict:
    """PCIe ceiling of the e2e number on this box: the step's H2D and D2H
    bytes copied between pinned host memory and the device on two streams
    concurrently (no kernel), best of 3; GDOF/s if transfers were all."""
    import torch

    hin = torch.empty(h2d // 8, dtype=torch.float64, pin_memory=True)
    hout = torch.empty(d2h // 8, dtype=torch.float64, pin_memory=True)
    din = torch.empty(h2d // 8, dtype=torch.float64, device="cuda")
    dout = torch.empty(d2h // 8, dtype=torch.float64, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    best = {}
    for mode in ("h2d", "d2h", "both"):
        ts = []
        for _ in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            if mode in ("h2d", "both"):
                with torch.cuda.stream(s1):
                    din.copy_(hin, non_blocking=True)
            if mode in ("d2h", "both"):
                with torch.cuda.stream(s2):
                    hout.copy_(dout, non_blocking=True)
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        best[mode] = min(ts)
    del hin, hout, din, dout
    return {"h2d_gbs": round(h2d / best["h2d"] / 1e9, 1), "d2h_gbs": round(d2h / best["d2h"] / 1e9, 1),
            "concurrent_ms": round(best["both"] * 1e3, 3), "gdof_s": ndof / best["both"] / 1e9}


def run_sweep(args, ws, rank, dist, clk, quick=False):
    """Every cell: a block of >= 1 GB algorithmic traffic per apply built from
    a tiled pool of seeded elements, timed over >= 0.15 s of back-to-back
    applies with CUDA events (max over ranks), parity of 6 sampled elements
    against the CPU oracle on identical inputs, clocks over the cell's
    window."""
    import torch

    import oracle as O
    import paper_2604_04644_b200 as sk
    from oracle.geom import deformed_coords
    from paper_2604_04644_b200.geometry import synthetic_affine_vertices, synthetic_deformation_params

    peaks, _ = _peaks()
    hbm, fp64 = peaks.get("hbm_gbs", 6650.0), _fp64_peak()
    kinds = {"helm": (sk.OperatorKind.HELMHOLTZ_COLL, 1.0), "stiff": (sk.OperatorKind.HELMHOLTZ_COLL, 0.0),
             "mass": (sk.OperatorKind.MASS, 1.0), "helmp": (sk.OperatorKind.HELMHOLTZ_COLL, 1.0)}
    params = synthetic_deformation_params(POOL, SEED)
    verts = {}
    rng = np.random.default_rng(1234 + rank)
    res = []
    cell_bytes = args.sweep_gb * 1e9
    for tab, op, deformed, s, P in _cells(quick, args.sweep_tables.split(",") if args.sweep_tables else None):
        kind, lam = kinds[op]
        shp = sk.Shape(s)
        b = sk.build_shape_basis(shp, P)
        bel = sk.operator_bytes(kind, shp, P, deformed, lam)
        if deformed:
            E = max(POOL, int(cell_bytes / bel))
            reps_e = -(-E // POOL)
            fac = sk.GeometricFactors(sk.GeometryClass.DEFORMED, shp, E, params=np.tile(params, (reps_e, 1))[:E], basis=b)
        else:
            # regular geometry is FP64-bound (7 doubles per element): size by work
            E = int(min(1 << 21, max(POOL, 4e10 / sk.operator_flops(kind, shp, P))))
            if s not in verts:
                verts[s] = synthetic_affine_vertices(shp, POOL, SEED)
            pool = sk.make_affine_block(shp, verts[s])
            reps_e = -(-E // POOL)
            fac = sk.GeometricFactors(sk.GeometryClass.REGULAR, shp, E,
                                      dxi_dx=np.tile(pool.dxi_dx, (reps_e, 1, 1))[:E],
                                      jac=np.tile(pool.jac, reps_e)[:E])
        blk = sk.Block(b, fac, sk.FieldState.COEFF, 1, 1)
        xd = blk.device(sk.AccessQualifier.WRITE_ONLY)
        gen = torch.Generator(device=xd.device)
        gen.manual_seed(P * 100 + SHAPES.index(s))
        xd.uniform_(-1.0, 1.0, generator=gen)
        out = blk.like(sk.FieldState.COEFF)
        if op == "mass":
            fn = lambda: sk.mass_apply(blk, out=out)  # noqa: E731
        elif op == "helmp":  # metric recomputed per chunk from the 12 parameters per element
            fn = lambda: sk.helmholtz_apply_params(blk, lam, out=out, check=False)  # noqa: E731
        else:
            fn = lambda: sk.helmholtz_apply(blk, lam, out=out)  # noqa: E731
        fn()
        torch.cuda.synchronize()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record()
        fn()
        t1.record()
        torch.cuda.synchronize()
        est = max(t0.elapsed_time(t1) / 1e3, 1e-6)
        reps = int(min(400, max(5, 0.15 / est)))
        if dist:
            rt = torch.tensor([reps], device="cuda")
            dist.all_reduce(rt, op=dist.ReduceOp.MAX)
            reps = int(rt.item())
            dist.barrier()
        torch.cuda.synchronize()
        w0 = time.perf_counter()
        t0.record()
        for _ in range(reps):
            fn()
        t1.record()
        torch.cuda.synchronize()
        w1 = time.perf_counter()
        ms = t0.elapsed_time(t1) / reps
        # parity on sampled elements, identical inputs, CPU oracle
        err = None
        if rank == 0:
            idx = sorted({0, 1, E // 2, E - 2, E - 1, int(rng.integers(0, E))})
            el = O.element(s, P)
            nm = b.n_modes
            xs = xd.view(E, nm)[idx].cpu().numpy().T
            ys = out.device(sk.AccessQualifier.READ_ONLY).view(E, nm)[idx].cpu().numpy().T
            if deformed:
                prm = params[[i % POOL for i in idx]]
                geo = O.deformed_geometry_from_coords(el, deformed_coords(el, prm))
            else:
                geo = O.affine_geometry(s, verts[s][[i % POOL for i in idx]])
            ref = O.mass(el, geo, xs) if op == "mass" else O.helmholtz_coll(el, geo, xs, lam)
            err = O.rel_diff(ys, ref)
        del blk, out, fac, xd
        torch.cuda.empty_cache()
        res.append((tab, s, P, E, ms, err, clk.summary(w0, w1) if clk else None, kind, lam, deformed))
    # max over ranks of every cell's time (weak scaling: each rank ran its own block)
    times = torch.tensor([r[4] for r in res], dtype=torch.float64, device="cuda")
    if dist:
        dist.all_reduce(times, op=dist.ReduceOp.MAX)
    tables: dict = {}
    info: dict = {}
    for r, ms in zip(res, times.tolist()):
        tab, s, P, E, _, err, ck, kind, lam, deformed = r
        shp = sk.Shape(s)
        nm = sk.mode_count(shp, P)
        bel = sk.operator_bytes(kind, shp, P, deformed, lam)
        if tab == "helm_recompute":
            bel = 8 * (2 * nm + 12)  # modes in/out + 12 deformation parameters
        fl = sk.operator_flops(kind, shp, P)
        gdof = ws * nm * E / (ms / 1e3) / 1e9
        roof_hbm = ws * hbm * 1e9 / bel * nm / 1e9
        roof_fp = ws * fp64 * 1e12 / fl * nm / 1e9
        roof = min(roof_hbm, roof_fp)
        frac = gdof / roof
        row = [P, float(f"{gdof:.4g}"), round(frac, 3), None if err is None else float(f"{err:.1e}"),
               None if not ck or ck["sm_mhz"] is None else round(ck["sm_mhz"])]
        tables.setdefault(tab, {}).setdefault(s, []).append(row)
        meta = info.setdefault(tab, {"bound": set(), "throttle": set(), "max_parity": 0.0})
        meta["bound"].add("hbm" if roof_hbm <= roof_fp else "fp64")
        meta["throttle"].update(ck["reasons"] if ck else [])
        meta["max_parity"] = max(meta["max_parity"], err or 0.0)
    # hex / tet DOF/s per order, streamed and recomputed metric
    for tab in ("helm_deformed", "helm_recompute"):
        t = tables.get(tab, {})
        if "hex" in t and "tet" in t:
            tet = {r[0]: r[1] for r in t["tet"]}
            info[tab]["hex_over_tet"] = {str(r[0]): round(r[1] / tet[r[0]], 2) for r in t["hex"] if r[0] in tet}
    for tab, meta in info.items():
        if "hex_over_tet" in meta:
            tables[tab]["hex_over_tet"] = meta["hex_over_tet"]
        tables[tab]["bound"] = sorted(meta["bound"])
        tables[tab]["throttle"] = sorted(meta["throttle"])
        tables[tab]["max_parity"] = float(f"{meta['max_parity']:.1e}")
    return tables, fp64


def _sample_parity(blocks, outs, spec, rank, n_extra=2):
    """Max-normalised error (speckern bench.py:192-194) of the timed outputs
    on sampled elements of every block -- first, middle, last and random
    ones -- against the CPU oracle on identical inputs (the same seeded
    geometry, the device-resident coefficients)."""
    import oracle as O
    import paper_2604_04644_b200 as sk
    from oracle.geom import deformed_coords

    rng = np.random.default_rng(99)
    worst = 0.0
    for k, ((shape, P, E), blk, out) in enumerate(zip(spec, blocks, outs)):
        idx = sorted({0, 1, E // 2, E - 2, E - 1, *[int(v) for v in rng.integers(0, E, n_extra)]})
        idx = [i for i in idx if 0 <= i < E]
        el = O.element(shape, P)
        nm = blk.basis.n_modes
        xs = blk.device(sk.AccessQualifier.READ_ONLY).view(E, nm)[idx].cpu().numpy().T
        ys = out.device(sk.AccessQualifier.READ_ONLY).view(E, nm)[idx].cpu().numpy().T
        prm = np.concatenate([O.deformation_params(1, SEED + k, first=rank * E + i) for i in idx])
        geo = O.deformed_geometry_from_coords(el, deformed_coords(el, prm))
        worst = max(worst, O.rel_diff(ys, O.helmholtz_coll(el, geo, xs, LAM)))
    return {"max_rel_err": float(f"{worst:.2e}"), "elements_checked_per_block": len(idx),
            "metric": "max-normalised vs CPU oracle (speckern bench.py:192-194)"}


def run_device(args, ws, rank, local):
    import torch

    import paper_2604_04644_b200 as sk
    from paper_2604_04644_b200 import _lib
    import oracle as O

    # SK_BENCH_SHARE_GPU=1: every rank on cuda:0 over gloo -- a functional
    # check of the multi-rank code path on a one-GPU box (timings meaningless)
    share = os.environ.get("SK_BENCH_SHARE_GPU") == "1"
    torch.cuda.set_device(0 if share else local)
    dist = None
    if ws > 1:
        import torch.distributed as dist

        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        chk = torch.ones(1, device="cuda")
        dist.all_reduce(chk)  # communicator up: comm_nranks == world size
        assert int(chk.item()) == ws, "communicator does not span every rank"
    dev = torch.cuda.current_device()
    clk = Clocks(dev).start()  # sampling from before the warm-up on
    wl = WORKLOADS[args.workload]
    spec = [(s, P, args.elements or e) for s, P, e in wl["blocks"]]
    if args.workload in ("c0hex", "c0prism", "c0tet", "c0pyr"):
        return run_c0(args, ws, rank, dist, dev, wl, clk)

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
    cold = args.workload == "hex4"  # L2-resident workload: flush L2 before every timed apply
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda") if cold else None
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(nb + 1)] for _ in range(args.steps)]

    def step(marks=None):
        if flush is not None:
            flush.zero_()
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
    torch.cuda.synchronize()
    w0 = time.perf_counter()
    t0.record(stream)
    for i in range(args.steps):
        step(ev[i])
    t1.record(stream)
    torch.cuda.synchronize()
    w1 = time.perf_counter()
    launches = _lib.launch_count() - n0
    if dist:
        dist.barrier()
    ms = t0.elapsed_time(t1)
    per_block_ms = [sum(ev[i][b].elapsed_time(ev[i][b + 1]) for i in range(args.steps)) / args.steps for b in range(nb)]
    if cold:  # the apply itself (cold L2), not the flush kernel
        ms = sum(per_block_ms) * args.steps
    tmax = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if dist:
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
    ms_max = float(tmax.item())
    ndof_rank = sum(b.basis.n_modes * b.n_elements for b in blocks)
    ndof = ndof_rank * ws
    value = ndof * args.steps / (ms_max / 1e3) / 1e9
    main_clocks = clk.summary(w0, w1)
    parity = _sample_parity(blocks, outs, spec, rank) if rank == 0 else None

    warm_us = None
    if cold:
        # L2-warm latency of the same apply, CUDA-graph captured back to back
        g = torch.cuda.CUDAGraph()
        s2 = torch.cuda.Stream()
        s2.wait_stream(stream)
        with torch.cuda.stream(s2):
            for _ in range(3):
                sk.helmholtz_apply(blocks[0], LAM, out=outs[0])
            with torch.cuda.graph(g, stream=s2):
                for _ in range(20):
                    sk.helmholtz_apply(blocks[0], LAM, out=outs[0])
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        a, c = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(10):
            g.replay()
        c.record()
        torch.cuda.synchronize()
        warm_us = a.elapsed_time(c) / 200 * 1e3

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
    e0 = time.perf_counter()
    for _ in range(e2e_steps):
        for blk, out in zip(blocks, outs):
            blk.host(sk.AccessQualifier.READ_WRITE)  # host copy is now the live one
            sk.helmholtz_apply(blk, LAM, out=out)  # -> H2D transfer + kernel
            out.host()  # -> D2H transfer of the result
    torch.cuda.synchronize()
    we = torch.tensor([time.perf_counter() - e0], dtype=torch.float64, device="cuda")
    if dist:
        dist.all_reduce(we, op=dist.ReduceOp.MAX)
    e2e_val = ndof * e2e_steps / float(we.item()) / 1e9
    copy_bound = _copy_ceiling(h2d, d2h, ndof)

    # roofline of the dominant kernel: algorithmic bytes per launch / its
    # average duration (CUDA events on the launching stream)
    peaks, src = _peaks()
    hbm = peaks.get("hbm_gbs", 6650.0)
    dom = int(np.argmax(per_block_ms))
    db = blocks[dom]
    bytes_per_launch = sk.operator_bytes(sk.OperatorKind.HELMHOLTZ_COLL, db.shape, db.basis.order, True, LAM) * db.n_elements
    achieved = bytes_per_launch / (per_block_ms[dom] / 1e3) / 1e9
    step_bytes = sum(sk.operator_bytes(sk.OperatorKind.HELMHOLTZ_COLL, b.shape, b.basis.order, True, LAM) * b.n_elements
                     for b in blocks)
    traffic = None
    prof = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(prof) and not cold:
        try:
            with open(prof) as fh:
                per_el = json.load(fh).get(f"{db.shape.value}_P{db.basis.order}_helm_per_element_bytes")
            traffic = per_el * db.n_elements if per_el else None
        except (OSError, ValueError):
            traffic = None

    # the BASELINE metric table (every shape x P), default workload only
    sweep = args.sweep == "on" or (args.sweep == "auto" and args.workload == "tet4")
    tables = fp64 = None
    if sweep:
        sw0 = time.perf_counter()
        tables, fp64 = run_sweep(args, ws, rank, dist, clk, quick=args.sweep_quick)
        sweep_s = time.perf_counter() - sw0

    cpu = None
    if rank == 0 and ws == 1:
        cores = os.cpu_count() or 1
        ref = CpuReference(cores, min(_per_core(spec), max(e for _, _, e in spec)), [(s, P) for s, P, _ in spec])
        reps = ref.calibrate(10.0)
        dofs, dt = ref.run(reps)
        ref.close()
        what = ("unmodified speckern (baseline/_ref) apply_operator(HELMHOLTZ_COLL, SUM_FAC)"
                if ref.kind == "reference" else "oracle port of speckern's sum-factorised Helmholtz")
        cpu = {
            "value": dofs / dt / 1e9,
            "unit": UNIT,
            "cores": cores,
            "kind": ref.kind,
            "sample": f"{what}: {ref.per_core * cores} elements of the workload ({cores} processes x "
                      f"{ref.per_core}, blocks round-robin) x {reps} passes: {dofs / 1e6:.0f} MDOF in {dt:.1f} s",
        }
    clk.stop()
    if rank == 0:
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
                "peak": hbm,
                "unit": "GB/s",
                "frac": achieved / hbm,
                "traffic": traffic,
                "peak_source": src,
                "bytes_per_launch": bytes_per_launch,
                "kernel": f"helmholtz {db.shape.value} P={db.basis.order}",
                "step_frac": step_bytes / (ms / 1e3 / args.steps) / 1e9 / hbm,
            },
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "copy_bound": {**copy_bound, "frac": e2e_val / copy_bound["gdof_s"]}},
            "gpu_launches": launches,
            "clocks": main_clocks,
            "parity": parity,
            "comm": {"backend": dist.get_backend() if dist else None, "world": ws, "collectives_in_timed_region": 0},
        }
        if nb > 1:
            line["per_block_ms"] = {f"{b.shape.value}": m for b, m in zip(blocks, per_block_ms)}
        if warm_us is not None:
            line["latency_us"] = {"cold_l2": ms_max / args.steps * 1e3, "warm_l2_graph": warm_us}
        if tables is not None:
            line["per_shape_P"] = {
                "columns": ["P", "gdof_s", "roofline_frac", "parity_maxrel", "sm_mhz"],
                "roofline": f"min(HBM {hbm:.0f} GB/s x N_P / bytes_el, FP64 {fp64:.1f} TF x N_P / flops_el), "
                            "bytes_el = 8(2N_P + 7N_Q) (6N_Q stiffness, N_Q mass; 7 / 6 / 1 regular; "
                            "helm_recompute 8(2N_P + 12): metric rebuilt per chunk from 12 parameters), "
                            "flops_el = reference operator_flops",
                "parity": "6 sampled elements per cell vs CPU oracle, max-normalised (speckern bench.py:192-194)",
                "cells": f"deformed: max({POOL}, {args.sweep_gb:.1f} GB / bytes_el) elements per apply; regular: "
                         f"min(2^21, max({POOL}, 4e10 / flops_el)); tiled pool of {POOL} seeded elements; "
                         "time = CUDA events over >= 0.15 s of back-to-back applies",
                "seconds": round(sweep_s, 1),
                **tables,
            }
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def run_c0(args, ws, rank, dist, dev, wl, clk):
    """Assembled C0 Helmholtz: gather -> elemental kernel -> scatter -> NCCL
    exchange of the two shared DOF layers, all inside the timed region."""
    import torch

    from paper_2604_04644_b200 import _lib
    from paper_2604_04644_b200.assembly import C0HexMesh, C0PrismMesh

    P = 4
    prism = args.workload == "c0prism"
    tet = args.workload in ("c0tet", "c0pyr")  # cube meshes with level-ordered DOFs
    if tet:
        from paper_2604_04644_b200.assembly import C0PyrMesh, C0TetMesh

        n = 40 if not args.elements else max(1, round((args.elements / 6) ** (1.0 / 3.0)))
        cls = C0TetMesh if args.workload == "c0tet" else C0PyrMesh
        mesh = cls(n, n, n * ws, P, rank=rank, world=ws)
    elif prism:
        n = 48 if not args.elements else max(1, round((args.elements / 2) ** (1.0 / 3.0)))
        mesh = C0PrismMesh(n, n, n * ws, P, rank=rank, world=ws)
    else:
        n = 64 if not args.elements else max(1, round(args.elements ** (1.0 / 3.0)))
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
    torch.cuda.synchronize()
    w0 = time.perf_counter()
    t0.record(stream)
    for _ in range(args.steps):
        mesh.helmholtz(x, LAM)
    t1.record(stream)
    torch.cuda.synchronize()
    w1 = time.perf_counter()
    launches = _lib.launch_count() - n0
    ms = t0.elapsed_time(t1)
    tmax = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if dist:
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
    ms_max = float(tmax.item())
    if tet:  # plane + between-level DOFs per cube layer, plus the last plane
        n_global = (mesh.n_dofs - mesh.layer) // mesh.nzl * (n * ws) + mesh.layer
    else:
        n_global = mesh.layer * (n * ws * P + 1)  # DOF layers along the slab axis
    value = n_global * args.steps / (ms_max / 1e3) / 1e9
    # e2e: host DOF vector in, host result out, every step
    xh = torch.empty(mesh.n_dofs, dtype=torch.float64).pin_memory().uniform_(-1.0, 1.0)
    yh = torch.empty_like(xh).pin_memory()
    e2e_steps = max(3, min(args.steps, 10))
    torch.cuda.synchronize()
    e0 = time.perf_counter()
    for _ in range(e2e_steps):
        yh.copy_(mesh.helmholtz(xh.to("cuda", non_blocking=True), LAM))
    torch.cuda.synchronize()
    we = torch.tensor([time.perf_counter() - e0], dtype=torch.float64, device="cuda")
    if dist:
        dist.all_reduce(we, op=dist.ReduceOp.MAX)
    e2e_val = n_global * e2e_steps / float(we.item()) / 1e9
    peaks, src = _peaks()
    import paper_2604_04644_b200 as sk

    shp = mesh.basis.shape
    bel = sk.operator_bytes(sk.OperatorKind.HELMHOLTZ_COLL, shp, P, True, LAM)
    step_bytes = bel * mesh.E + 2 * 8 * mesh.n_dofs
    achieved = step_bytes / (ms / 1e3 / args.steps) / 1e9
    clk.stop()
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
            "data": f"synthetic (conforming deformed {shp.value} mesh, device geometry builder)",
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
            "clocks": clk.summary(w0, w1),
            "comm": {"backend": dist.get_backend() if dist else None, "world": ws,
                     "collectives_in_timed_region": "2 P2P send/recv per interface per step" if ws > 1 else 0},
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def run_reference_sweep(args):
    """Reference CPU path per shape x order: one JSON line each, to sit beside
    the device sweep.  Bounded samples (~2 s per case)."""
    cores = os.cpu_count() or 1
    for shape in SHAPES:
        for P in range(2, 11):
            per_core = max(8, int(1024 * (5.0 / (P + 1)) ** 3))
            ref = CpuReference(cores, per_core, [(shape, P)])
            reps = ref.calibrate(1.5)
            vals = []
            for _ in range(3):
                dof, dt = ref.run(reps)
                vals.append(dof / dt / 1e9)
            ref.close()
            print(json.dumps({"impl": "reference", "op": "helm", "shape": shape, "P": P,
                              "gdof_s": statistics.median(vals), "cores": cores, "kind": ref.kind,
                              "sample": f"{per_core * cores} elements x {reps} passes, median of 3"}), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["sk", "reference"], default="sk")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="tet4")
    ap.add_argument("--elements", type=int, default=0, help="override elements per block per GPU")
    ap.add_argument("--sweep", choices=["auto", "on", "off"], default="auto",
                    help="per (shape, P) table in the JSON line (auto: default workload only)")
    ap.add_argument("--sweep-quick", action="store_true", help="P in {2,4,6,8,10} only")
    ap.add_argument("--sweep-gb", type=float, default=SWEEP_BYTES / 1e9,
                    help="algorithmic GB per apply per deformed cell (e.g. 100: max elements per GPU, configs[4])")
    ap.add_argument("--sweep-tables", default="", help="comma list of per_shape_P tables to run (default all)")
    ap.add_argument("--ref-sweep", action="store_true", help="with --impl reference: CPU GDOF/s per shape x order")
    args = ap.parse_args()
    if args.gpus < 1:
        raise SystemExit("--gpus must be >= 1")
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(_relaunch(args))
    ws, rank, local = _dist()
    if ws != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={ws}: launch one rank per GPU")
    if args.impl == "reference" and args.ref_sweep:
        if rank == 0:
            run_reference_sweep(args)
        return
    if args.impl == "reference":
        run_reference(args, ws, rank)
        return
    run_device(args, ws, rank, local)


if __name__ == "__main__":
    main()
