"""GPU mode of the reference bench harness and CLI (`cabl-bench`).

Counterpart of reference proj/include/cabl/bench.hpp:32-431 (SweepConfig,
run_config, run_sweep, CSV emit/parse, SVG) and proj/tools/bench_main.cpp
(flags, size ranges, exit codes), for the B200 kernels:

    python -m paper_2108_02025_b200.benchcli --kernel all --sizes 256:1048576:4 \\
        --threads 1,4 --reps 5 --dtype f64 --csv sweep.csv --svg sweep.svg

What stays from the reference:
  * kernels dot | ger | gemv-row | gemv-col | all; square matrices m = n =
    size, `dot` uses the size as the vector length (bench.hpp:126);
  * --sizes as a comma list or start:stop:factor (bench_main.cpp:36-57);
  * every configuration is spot-checked BEFORE timing and a mismatch aborts
    that configuration and makes the exit status 1 (bench.hpp:3-6, :183-189);
    errors exit 2 (bench_main.cpp:124-128);
  * flop accounting dot = 2n, gemv/ger = 2mn (bench.hpp:78-81);
  * CSV header `kernel,m,n,threads,reps,min_s,median_s,gflops,checksum`, 9
    significant digits, round-trips through parse_csv (bench.hpp:260-340);
  * SVG: log problem size vs GFLOP/s, one polyline per (kernel, threads).
What is new for the GPU: --dtype (the reference is fp64-only), --rect MxN
shapes, --gpus N (the sharded multi-GPU paths of SURVEY.md §8(e) through the
cabl_mgpu C ABI: DOT by chunks, GEMV row-major and GER by row blocks,
col-major GEMV by column blocks), CSV columns dtype, gbs, roofline_frac (of
the measured HBM peak x GPUs), gpus, layout; timing is CUDA events with the
L2 flushed between repetitions (GER also charged the write-back of the lines
it leaves dirty in L2); `threads` is validated against the descriptor (as the
reference does) and recorded, but does not shape the GPU launch.  The spot
check is an independent fp64 PyTorch computation on the device with the
reference's tolerances (dot and gemv: n*eps*sum|a_i b_i|), and for GER the
reference's bitwise rule (bench.hpp:139-146: ger == ger_ref, i.e. one fused
multiply-add per element): every element within one rounding of the exact
x_i*y_j + C_ij, and sampled elements equal to its correctly rounded value,
computed in exact rational arithmetic.
--bounds replaces the reference's CPU-cache bound columns (bench.hpp:214-226,
io_bounds.hpp:112-150 report()) by the HBM traffic model: alg_bytes (what
the operation must move), hbm_bound_s (that at the measured
peak), and — with --measure-dram — dram_bytes, the DRAM bytes ncu measured
for one call of each configuration (dram__bytes_read.sum +
dram__bytes_write.sum of the library's kernels in that call, cold L2), and
dram_per_alg = dram_bytes / alg_bytes (well above 1: re-reads).
"""
from __future__ import annotations

import argparse
import json
import math
import statistics
import sys
import zlib
from dataclasses import dataclass, field
from pathlib import Path

CSV_HEADER = "kernel,m,n,threads,reps,min_s,median_s,gflops,checksum"
CSV_GPU_SUFFIX = ",dtype,gbs,roofline_frac,gpus,layout"
CSV_GPU_SUFFIX_R1 = ",dtype,gbs,roofline_frac"  # round-1 documents still parse
# --bounds: the HBM traffic model in place of the reference's CPU-cache bound
# columns (reference bench.hpp:214-226, io_bounds.hpp report()): the bytes the
# operation must move, the time they take at the measured
# HBM peak — the B200 lower bound the measured median is compared against —
# and the DRAM bytes ncu measured (nan when not measured).
CSV_BOUNDS_SUFFIX = ",alg_bytes,hbm_bound_s,dram_bytes,dram_per_alg"
CSV_BOUNDS_SUFFIX_R1 = ",alg_bytes,hbm_bound_s"
KERNELS = ("dot", "ger", "gemv-row", "gemv-col")
LAYOUT = {"dot": "vector", "ger": "row-major", "gemv-row": "row-major", "gemv-col": "col-major"}


@dataclass
class BenchRecord:
    kernel: str
    m: int
    n: int
    threads: int = 1
    reps: int = 0
    min_s: float = 0.0
    median_s: float = 0.0
    gflops: float = 0.0
    checksum: float = 0.0
    dtype: str = "f64"
    gbs: float = 0.0
    roofline_frac: float = 0.0
    gpus: int = 1
    layout: str = ""
    alg_bytes: int | None = None      # --bounds
    hbm_bound_s: float | None = None  # --bounds
    dram_bytes: float = math.nan      # --bounds --measure-dram (ncu)
    dram_per_alg: float = math.nan


@dataclass
class SweepConfig:
    kernels: list = field(default_factory=lambda: list(KERNELS))
    sizes: list = field(default_factory=lambda: [256, 1024, 4096])
    rects: list = field(default_factory=list)  # extra (m, n) shapes for matrix kernels
    threads: list = field(default_factory=lambda: [1])
    reps: int = 5
    seed: int = 42
    dtype: str = "f64"
    max_threads: int = 8
    bounds: bool = False
    gpus: int = 1


# ------------------------------------------------------------------ parsing
def parse_sizes(spec: str) -> list[int]:
    if ":" in spec:
        parts = spec.split(":")
        if len(parts) != 3:
            raise ValueError("--sizes range spec must be start:stop:factor")
        start, stop, factor = (int(p) for p in parts)
        if start < 1 or factor < 2:
            raise ValueError("--sizes range needs start >= 1 and factor >= 2")
        out, s = [], start
        while s <= stop:
            out.append(s)
            s *= factor
        return out
    return [int(t) for t in spec.split(",") if t.strip()]


def parse_rects(spec: str) -> list[tuple[int, int]]:
    out = []
    for tok in spec.split(","):
        if tok.strip():
            m, n = tok.lower().split("x")
            out.append((int(m), int(n)))
    return out


def load_descriptor(path: str):
    """Flat JSON machine descriptor (reference descriptor_json.hpp:3-15);
    'gpu' = the live device's descriptor (machine.py)."""
    from . import machine
    if path == "gpu":
        return machine.gpu_machine(0)
    return machine.load_descriptor_file(path)


# ---------------------------------------------------------------------- CSV
def _g9(v: float) -> str:
    return f"{v:.9g}"


def emit_csv(records: list[BenchRecord]) -> str:
    if not records:
        raise ValueError("emit_csv: no records")
    bounds = records[0].alg_bytes is not None
    lines = [CSV_HEADER + CSV_GPU_SUFFIX + (CSV_BOUNDS_SUFFIX if bounds else "")]
    for r in records:
        f = [r.kernel, str(r.m), str(r.n), str(r.threads), str(r.reps), _g9(r.min_s),
             _g9(r.median_s), _g9(r.gflops), _g9(r.checksum), r.dtype, _g9(r.gbs),
             _g9(r.roofline_frac), str(r.gpus), r.layout or LAYOUT.get(r.kernel, "")]
        if bounds:
            f += [str(r.alg_bytes), _g9(r.hbm_bound_s), _g9(r.dram_bytes), _g9(r.dram_per_alg)]
        lines.append(",".join(f))
    return "\n".join(lines) + "\n"


def parse_csv(text: str) -> list[BenchRecord]:
    """Reads the documents emit_csv writes, round-1 GPU documents (no gpus /
    layout / dram columns) and the reference's own 9-column CSV."""
    rows = text.splitlines()
    if not rows:
        raise ValueError("parse_csv: empty document")
    forms = {CSV_HEADER: (9, False, False, False),
             CSV_HEADER + CSV_GPU_SUFFIX_R1: (12, True, False, False),
             CSV_HEADER + CSV_GPU_SUFFIX_R1 + CSV_BOUNDS_SUFFIX_R1: (14, True, False, True),
             CSV_HEADER + CSV_GPU_SUFFIX: (14, True, True, False),
             CSV_HEADER + CSV_GPU_SUFFIX + CSV_BOUNDS_SUFFIX: (18, True, True, True)}
    if rows[0] not in forms:
        raise ValueError("parse_csv: unexpected header")
    want, gpu, cols2, bounds = forms[rows[0]]
    out = []
    for line in rows[1:]:
        if not line:
            continue
        f = line.split(",")
        if len(f) != want:
            raise ValueError("parse_csv: bad field count")
        r = BenchRecord(f[0], int(f[1]), int(f[2]), int(f[3]), int(f[4]), float(f[5]),
                        float(f[6]), float(f[7]), float(f[8]))
        k = 9
        if gpu:
            r.dtype, r.gbs, r.roofline_frac = f[9], float(f[10]), float(f[11])
            k = 12
        if cols2:
            r.gpus, r.layout = int(f[12]), f[13]
            k = 14
        else:
            r.layout = LAYOUT.get(r.kernel, "")
        if bounds:
            r.alg_bytes, r.hbm_bound_s = int(f[k]), float(f[k + 1])
            if want == 18:
                r.dram_bytes, r.dram_per_alg = float(f[k + 2]), float(f[k + 3])
        out.append(r)
    return out


# ---------------------------------------------------------------------- SVG
def emit_svg(records: list[BenchRecord], metric: str = "gflops") -> str:
    if not records:
        raise ValueError("emit_svg: no records")
    series: dict[tuple[str, int], list[tuple[float, float]]] = {}
    for r in records:
        size = r.n if r.kernel == "dot" else r.m * r.n
        series.setdefault((r.kernel, r.threads), []).append(
            (math.log10(max(1.0, size)), getattr(r, metric)))
    xs = [p[0] for pts in series.values() for p in pts]
    ys = [p[1] for pts in series.values() for p in pts]
    x0, x1 = min(xs), max(xs)
    if x1 - x0 < 1e-9:
        x1 = x0 + 1.0
    ymax = max(max(ys), 1e-12) * 1.05
    W, H, L, R, T, B = 960, 560, 70, 240, 40, 60
    pw, ph = W - L - R, H - T - B
    px = lambda x: L + (x - x0) / (x1 - x0) * pw  # noqa: E731
    py = lambda y: T + ph - y / ymax * ph  # noqa: E731
    colors = ["#1f77b4", "#ff7f0e", "#2ca02c", "#d62728", "#9467bd", "#8c564b", "#e377c2",
              "#7f7f7f", "#bcbd22", "#17becf"]
    out = ['<?xml version="1.0" encoding="UTF-8"?>',
           f'<svg xmlns="http://www.w3.org/2000/svg" width="{W}" height="{H}" '
           f'viewBox="0 0 {W} {H}">',
           f'  <rect width="{W}" height="{H}" fill="white"/>',
           f'  <line x1="{L}" y1="{T + ph}" x2="{L + pw}" y2="{T + ph}" stroke="black"/>',
           f'  <line x1="{L}" y1="{T}" x2="{L}" y2="{T + ph}" stroke="black"/>']
    for k in range(math.ceil(x0), math.floor(x1) + 1):
        out.append(f'  <text x="{px(k):.1f}" y="{T + ph + 20}" font-size="12" '
                   f'text-anchor="middle">1e{k}</text>')
    for k in range(6):
        yv = ymax * k / 5
        out.append(f'  <text x="{L - 9}" y="{py(yv) + 4:.1f}" font-size="12" '
                   f'text-anchor="end">{_g9(yv)}</text>')
    label = {"gflops": "GFLOP/s", "gbs": "GB/s"}.get(metric, metric)
    out.append(f'  <text x="{L + pw / 2}" y="{H - 15}" font-size="13" text-anchor="middle">'
               f'problem size (elements, log)</text>')
    out.append(f'  <text x="18" y="{T + ph / 2}" font-size="13" text-anchor="middle" '
               f'transform="rotate(-90 18 {T + ph / 2})">{label} (B200)</text>')
    ly = T + 10
    for i, (key, pts) in enumerate(sorted(series.items())):
        pts.sort()
        col = colors[i % len(colors)]
        coords = " ".join(f"{px(x):.1f},{py(y):.1f}" for x, y in pts)
        out.append(f'  <polyline fill="none" stroke="{col}" stroke-width="2" points="{coords}"/>')
        out.append(f'  <text x="{L + pw + 20}" y="{ly + 4}" font-size="12" fill="{col}">'
                   f'{key[0]} (t={key[1]})</text>')
        ly += 18
    out.append("</svg>")
    return "\n".join(out) + "\n"


# -------------------------------------------------------------------- sweep
def _alg_bytes(kernel: str, m: int, n: int, s: int, gpus: int = 1) -> int:
    """x is read once per GPU for GEMV row blocks, y for GER;
    a col-major GEMV by column blocks reads its slice of x and its replica of c."""
    if kernel == "dot":
        return 2 * n * s
    if kernel == "gemv-row":
        return m * n * s + gpus * n * s + 2 * m * s
    if kernel == "gemv-col":
        return m * n * s + n * s + 2 * gpus * m * s
    return 2 * m * n * s + m * s + gpus * n * s


def _split(kernel: str, m: int, n: int, gpus: int) -> list[tuple[int, int]]:
    """The sharded dimension of each kernel, balanced contiguous ranges
    (reference parallel_chunks, thread_pool.hpp:153-164): DOT chunks of the
    vectors, GEMV row-major / GER row blocks, col-major GEMV column blocks."""
    from .mgpu import partition
    total = n if kernel in ("dot", "gemv-col") else m
    return [partition(total, gpus, r) for r in range(gpus)]


def _round_exact_f32(q):
    """The float32 nearest to the rational q (ties to even)."""
    import numpy as np
    f = np.float32(float(q))
    best = f
    for c in (np.nextafter(f, np.float32(-np.inf)), np.nextafter(f, np.float32(np.inf))):
        from fractions import Fraction
        d_c, d_b = abs(Fraction(float(c)) - q), abs(Fraction(float(best)) - q)
        if d_c < d_b or (d_c == d_b and (int(c.view(np.uint32)) & 1) == 0):
            best = c
    return best


def _ger_exact_sample(x, y, C0, C1, m, n, dtype, k=512, seed=0) -> str | None:
    """ger_ref's bits (one fused multiply-add per element) on k sampled
    elements plus the corners: C1(i,j) must be x_i*y_j + C0(i,j) correctly
    rounded, computed in exact rational arithmetic (reference bench.hpp:139-146
    compares ger with ger_ref bitwise)."""
    import random
    from fractions import Fraction
    rng = random.Random(seed)
    idx = {(0, 0), (m - 1, n - 1), (0, n - 1), (m - 1, 0)}
    while len(idx) < min(k + 4, m * n):
        idx.add((rng.randrange(m), rng.randrange(n)))
    ii = sorted(idx)
    import torch
    rows = torch.tensor([i for i, _ in ii], device=C1.device)
    cols = torch.tensor([j for _, j in ii], device=C1.device)
    flat = rows * n + cols
    xs, ys = x[rows].double().tolist(), y[cols].double().tolist()
    c0s, c1s = C0[flat].double().tolist(), C1[flat].double().tolist()
    for (i, j), xv, yv, cv, got in zip(ii, xs, ys, c0s, c1s):
        q = Fraction(xv) * Fraction(yv) + Fraction(cv)
        want = float(q) if dtype == torch.float64 else float(_round_exact_f32(q))
        if got != want:
            return f"C({i},{j}) = {got!r}, fma(x_i, y_j, C_ij) = {want!r}"
    return None


def _inputs(kernel, m, n, G, dt, seed, devs):
    """Seeded shard inputs on their devices (global counters, so the union of
    the shards is the one-GPU problem)."""
    import torch

    from . import cabl

    def fill(k, st, dev, off=0):
        return cabl.fill_uniform(torch.empty(k, dtype=dt, device=dev), seed, st, off)
    sh = []
    for r, (b, e) in enumerate(_split(kernel, m, n, G)):
        d = devs[r]
        if kernel == "dot":
            sh.append({"x": fill(e - b, 1, d, b), "y": fill(e - b, 2, d, b)})
        elif kernel == "ger":
            C0 = fill((e - b) * n, 5, d, b * n)
            sh.append({"x": fill(e - b, 1, d, b), "y": fill(n, 2, d), "C0": C0,
                       "C": cabl.DenseMatrix.wrap(C0.clone(), e - b, n, cabl.Layout.RowMajor)})
        elif kernel == "gemv-row":
            A = fill((e - b) * n, 3, d, b * n)
            c0 = fill(e - b, 4, d, b)
            sh.append({"A": cabl.DenseMatrix.wrap(A, e - b, n, cabl.Layout.RowMajor),
                       "x": fill(n, 1, d), "c0": c0, "c": c0.clone()})
        else:
            A = fill(m * (e - b), 3, d, b * m)
            c0 = fill(m, 4, d)
            sh.append({"A": cabl.DenseMatrix.wrap(A, m, e - b, cabl.Layout.ColMajor),
                       "x": fill(e - b, 1, d, b), "c0": c0, "c": c0.clone()})
    return sh


def _check(kernel, sh, m, n, dt, result) -> str | None:
    """Spot check of one call against fp64 PyTorch (reference tolerances) and,
    for GER, the exact-rounding rule."""
    import torch
    eps = float(torch.finfo(dt).eps)
    if kernel == "dot":
        want = sum(float((s["x"].double() * s["y"].double()).sum()) for s in sh)
        sumabs = sum(float((s["x"].double() * s["y"].double()).abs().sum()) for s in sh)
        if abs(result - want) > n * eps * sumabs + 4 * eps * abs(want):
            return f"abs diff = {abs(result - want):.3e}"
        return None
    if kernel == "ger":
        for s in sh:
            mr = s["x"].numel()
            if mr == 0:
                continue
            prod = s["x"].double()[:, None] * s["y"].double()[None, :]
            exact = s["C0"].double().view(mr, n) + prod
            got = s["C"].data.double().view(mr, n)
            tol = eps * (s["C0"].double().view(mr, n).abs() + prod.abs()) + torch.finfo(dt).tiny
            if not bool(((got - exact).abs() <= tol).all()):
                return "not within one rounding of x_i*y_j + C_ij"
            bad = _ger_exact_sample(s["x"], s["y"], s["C0"], s["C"].data, mr, n, dt)
            if bad:
                return "not bitwise ger_ref (one fma per element): " + bad
        return None
    if kernel == "gemv-row":
        for s in sh:
            mr = s["c"].numel()
            if mr == 0:
                continue
            A2 = s["A"].data.double().view(mr, n)
            want = s["c0"].double() + A2 @ s["x"].double()
            rowabs = A2.abs() @ s["x"].double().abs()
            err = (s["c"].double() - want).abs()
            if not bool((err <= n * eps * rowabs + 4 * eps * want.abs()).all()):
                return f"max abs diff = {float(err.max()):.3e}"
        return None
    want = sh[0]["c0"].double().cpu()
    rowabs = torch.zeros(m, dtype=torch.float64)
    for s in sh:
        k = s["x"].numel()
        A2 = s["A"].data.double().view(k, m).t()
        want = want + (A2 @ s["x"].double()).cpu()
        rowabs = rowabs + (A2.abs() @ s["x"].double().abs()).cpu()
    for s in sh:
        err = (s["c"].double().cpu() - want).abs()
        if not bool((err <= n * eps * rowabs + 4 * eps * want.abs()).all()):
            return f"max abs diff = {float(err.max()):.3e}"
    return None


def _caller(kernel, sh, pol, mg, dt, devs):
    """The call under test: the single-GPU API (mg None) or the cabl_mgpu C
    ABI over the shards.  Returns a thunk that runs one call and returns its
    DOT value (None for the matrix kernels)."""
    import torch

    from . import cabl
    if mg is None:
        s0 = sh[0]
        if kernel == "dot":  # no host read inside the call: the value is read after
            out1 = torch.empty(1, dtype=dt, device=devs[0])
            return lambda: (cabl.dot_into(s0["x"], s0["y"], 0.0, out1, pol), out1)[1]
        if kernel == "ger":
            return lambda: cabl.ger(s0["x"], s0["y"], s0["C"], pol)
        f = cabl.gemv_row_major if kernel == "gemv-row" else cabl.gemv_col_major
        return lambda: f(s0["A"], s0["x"], s0["c"], pol)
    xs = [s["x"] for s in sh]
    if kernel == "dot":
        ys = [s["y"] for s in sh]
        return lambda: mg.dot(xs, ys, 0.0, pol)
    if kernel == "ger":
        ys, Cs = [s["y"] for s in sh], [s["C"] for s in sh]
        return lambda: mg.ger_rm(xs, ys, Cs, pol)
    As, cs = [s["A"] for s in sh], [s["c"] for s in sh]
    if kernel == "gemv-row":
        return lambda: mg.gemv_rm(As, xs, cs, pol)
    return lambda: mg.gemv_cm_cols(As, xs, cs, pol)


def run_config(kernel: str, m: int, n: int, threads: int, cfg: SweepConfig, flush, peak: float,
               failures: list[str], mg=None, nvtx: bool = False) -> BenchRecord | None:
    """One configuration: seeded shard inputs, one call spot-checked against
    fp64 (a mismatch aborts the configuration, bench.hpp:183-189), then
    cfg.reps timed calls with the L2 of every device flushed before each.
    Device time: CUDA events on the stream(s) the call runs on; with several
    GPUs the max over devices.  nvtx: the --dram-pass mode — one more call
    between two marker kernels, untimed (measure_dram cuts the ncu list there)."""
    import torch

    from . import cabl
    dt = torch.float32 if cfg.dtype == "f32" else torch.float64
    s = 4 if cfg.dtype == "f32" else 8
    G = mg.size if mg is not None else 1
    devs = list(mg.devices) if mg is not None else [torch.cuda.current_device()]
    pol = cabl.ExecPolicy(cabl.derive_blocking_plan(cabl.default_machine(cfg.max_threads)), threads)
    salt = zlib.crc32(kernel.encode()) * 1000003 + m * 31 + n  # stable across processes
    sh = _inputs(kernel, m, n, G, dt, cfg.seed + salt, devs)
    rec = BenchRecord(kernel, 0 if kernel == "dot" else m, n, threads, cfg.reps, dtype=cfg.dtype,
                      gpus=G, layout=LAYOUT[kernel])
    call = _caller(kernel, sh, pol, mg, dt, devs)
    got = call()
    for d in devs:
        torch.cuda.synchronize(d)
    if kernel == "dot" and mg is None:
        got = float(got[0])
    fail = _check(kernel, sh, m, n, dt, got)
    if kernel == "dot":
        rec.checksum = got
    elif kernel == "ger":
        rec.checksum = sum(float(x["C"].data.double().sum()) for x in sh)
    else:
        rec.checksum = sum(float(x["c"].double().sum()) for x in sh) if kernel == "gemv-row" \
            else float(sh[0]["c"].double().sum())
    if fail:
        failures.append(f"kernel={kernel} m={rec.m} n={n} threads={threads} gpus={G}: "
                        f"oracle mismatch, {fail}")
        return None
    if nvtx:
        # the --dram-pass: one call between two marker kernels (torch's spin
        # kernel), so the ncu launch list can be cut into configurations
        for d in devs:
            torch.cuda.synchronize(d)
        torch.cuda._sleep(1)
        call()
        torch.cuda._sleep(1)
        for d in devs:
            torch.cuda.synchronize(d)
        return rec
    call()  # warm-up
    writes = kernel == "ger"  # charge the write-back of the lines C left dirty in L2
    times = []
    for _ in range(cfg.reps):
        flush()
        if mg is None:
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            call()
            if writes:
                flush.evict(devs[0])
            b.record()
            torch.cuda.synchronize(devs[0])
            t = a.elapsed_time(b) / 1e3
        else:
            # the C ABI call is synchronous; its device time per rank comes from
            # the library's own events (cabl_mgpu_last_call_ms), max over ranks
            call()
            t = max(mg.last_call_ms()) / 1e3
            if writes:  # the eviction pass after the call, per device, max
                ev = []
                for d in devs:
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    with torch.cuda.device(d):
                        a.record()
                        flush.evict(d)
                        b.record()
                    ev.append((a, b))
                for d in devs:
                    torch.cuda.synchronize(d)
                t += max(a.elapsed_time(b) for a, b in ev) / 1e3
        times.append(t - (flush.evict_s() if writes else 0.0))
    rec.min_s = max(min(times), 1e-12)
    rec.median_s = max(statistics.median(times), 1e-12)
    flops = 2 * n if kernel == "dot" else 2 * m * n
    rec.gflops = flops / rec.median_s / 1e9
    alg = _alg_bytes(kernel, m, n, s, G)
    rec.gbs = alg / rec.median_s / 1e9
    rec.roofline_frac = rec.gbs / (peak * G)
    if cfg.bounds:
        rec.alg_bytes = alg
        rec.hbm_bound_s = alg / (peak * G * 1e9)
    return rec


class _Flush:
    """L2 flush of every device in use (512 MiB write, then 512 MiB read: > L2,
    no dirty lines left), and the eviction pass that charges a writing
    kernel's deferred write-back (bench.py L2Flush.evict_)."""

    def __init__(self, devs):
        import torch
        self.bufs = {d: (torch.empty(128 << 20, dtype=torch.float32, device=d),
                         torch.zeros(128 << 20, dtype=torch.float32, device=d),
                         torch.zeros(64 << 20, dtype=torch.float32, device=d)) for d in devs}
        self._evict = None
        self.sync = False  # set for the cabl_mgpu path (its streams do not wait on torch's)

    def __call__(self):
        import torch
        for d, (w, r, _) in self.bufs.items():
            with torch.cuda.device(d):
                w.zero_()
                r.sum()
        # one device: stream order is enough, and leaving the flush running
        # hides the host's call overhead from the next call's events (a
        # synchronize here put ~15 us of Python + ctypes inside them); several
        # devices: the cabl_mgpu streams do not wait on torch's
        if len(self.bufs) > 1 or self.sync:
            for d in self.bufs:
                torch.cuda.synchronize(d)

    def evict(self, d):
        self.bufs[d][2].sum()

    def evict_s(self) -> float:
        import torch
        if self._evict is None:
            ts = []
            d = next(iter(self.bufs))
            for i in range(12):
                self()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                with torch.cuda.device(d):
                    a.record()
                    self.evict(d)
                    b.record()
                torch.cuda.synchronize(d)
                if i >= 2:
                    ts.append(a.elapsed_time(b) / 1e3)
            self._evict = sum(ts) / len(ts)
        return self._evict


def run_sweep(cfg: SweepConfig, nvtx: bool = False,
              use_mgpu: bool = False) -> tuple[list[BenchRecord], list[str]]:
    import torch
    if cfg.reps < 3:
        raise ValueError("run_sweep: repetitions must be >= 3")
    if not cfg.kernels or not (cfg.sizes or cfg.rects) or not cfg.threads:
        raise ValueError("run_sweep: kernels, sizes and threads must be non-empty")
    for k in cfg.kernels:
        if k not in KERNELS:
            raise ValueError(f"run_sweep: unknown kernel '{k}'")
    if any(s < 1 for s in cfg.sizes):
        raise ValueError("run_sweep: sizes must be >= 1")
    if any(t < 1 or t > cfg.max_threads for t in cfg.threads):
        raise ValueError("run_sweep: thread count out of range for this machine")
    if cfg.gpus < 1:
        raise ValueError("run_sweep: --gpus must be >= 1")
    if not torch.cuda.is_available():
        raise RuntimeError("no CUDA device (the B200 bench has no CPU path)")
    if torch.cuda.device_count() < cfg.gpus:
        raise RuntimeError(f"--gpus {cfg.gpus}: only {torch.cuda.device_count()} GPU(s) visible")
    peak = _peak()
    mg = None
    if cfg.gpus > 1 or use_mgpu:
        from .mgpu import MultiGpu
        mg = MultiGpu(list(range(cfg.gpus)))
    devs = list(range(cfg.gpus)) if mg is not None else [torch.cuda.current_device()]
    flush = _Flush(devs)
    flush.sync = mg is not None
    records, failures = [], []
    try:
        for k in cfg.kernels:
            shapes = [(s, s) for s in cfg.sizes] + ([] if k == "dot" else list(cfg.rects))
            for m, n in shapes:
                for t in cfg.threads:
                    r = run_config(k, m, n, t, cfg, flush, peak, failures, mg=mg, nvtx=nvtx)
                    if r is not None:
                        records.append(r)
    finally:
        if mg is not None:
            mg.close()
    return records, failures


def measure_dram(argv: list[str], records: list[BenchRecord], workdir: Path) -> None:
    """Fill dram_bytes / dram_per_alg from ncu: the same sweep re-run in
    --dram-pass mode (one call per configuration between two marker kernels),
    first plainly (it must exit 0 before ncu touches it), then under
    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum restricted to the
    markers and the library's kernels (namespace cabl_dev); the bytes of the
    library kernels between each pair of markers are the configuration's
    (cold L2: ncu flushes caches before every kernel)."""
    import csv
    import os
    import shutil
    import subprocess
    ncu = shutil.which("ncu") or "/usr/local/cuda/bin/ncu"
    base = [sys.executable, "-m", "paper_2108_02025_b200.benchcli", *argv, "--dram-pass"]
    env = dict(os.environ)
    r = subprocess.run(base, capture_output=True, text=True, env=env)
    if r.returncode != 0:
        raise RuntimeError(f"--measure-dram: the plain dram pass failed: {r.stderr[-400:]}")
    log = workdir / "cabl_dram_ncu.csv"
    cmd = [ncu, "--kernel-name-base", "demangled", "-k", "regex:spin_kernel|cabl_dev", "--metrics",
           "dram__bytes_read.sum,dram__bytes_write.sum", "--clock-control", "none", "--csv",
           "--log-file", str(log), *base]
    r = subprocess.run(cmd, capture_output=True, text=True, env=env)
    if r.returncode != 0 or not log.exists():
        raise RuntimeError(f"--measure-dram: ncu failed (rc {r.returncode}): "
                           f"{(r.stderr or r.stdout)[-400:]}")
    rows = list(csv.reader(log.read_text().splitlines()))
    hi = next(i for i, row in enumerate(rows) if row and row[0] == "ID")
    h = {k: j for j, k in enumerate(rows[hi])}
    launches: dict[int, list] = {}  # ID -> [name, bytes]
    for row in rows[hi + 1:]:
        if len(row) < len(h):
            continue
        lid = int(row[h["ID"]])
        unit = row[h["Metric Unit"]] if "Metric Unit" in h else "byte"
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
        ent = launches.setdefault(lid, [row[h["Kernel Name"]], 0.0])
        ent[1] += float(row[h["Metric Value"]].replace(",", "")) * scale
    totals: list[float] = []
    inside, acc = False, 0.0
    for lid in sorted(launches):
        name, b = launches[lid]
        if "spin_kernel" in name:
            if inside:
                totals.append(acc)
            inside, acc = not inside, 0.0
        elif inside:
            acc += b
    if len(totals) != len(records):
        raise RuntimeError(f"--measure-dram: {len(totals)} marked calls in the ncu list for "
                           f"{len(records)} configurations")
    for rec, t in zip(records, totals):
        rec.dram_bytes = t
        rec.dram_per_alg = t / rec.alg_bytes if rec.alg_bytes else math.nan


def _peak() -> float:
    p = Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json"
    if p.exists():
        return float(json.loads(p.read_text())["hbm_gbs"])
    return 6650.0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="cabl-bench (B200)",
                                 description="cache-aware level-1/2 kernel benchmark, GPU mode")
    ap.add_argument("--machine", default=None,
                    help="machine descriptor JSON, or 'gpu' for the live device (default: built-in)")
    ap.add_argument("--describe", action="store_true",
                    help="print the live GPU's machine descriptor JSON and exit")
    ap.add_argument("--kernel", default="all", choices=list(KERNELS) + ["all"])
    ap.add_argument("--sizes", default="256,1024,4096,16384")
    ap.add_argument("--rect", default="", help="extra MxN shapes for matrix kernels, e.g. 256x1048576")
    ap.add_argument("--threads", default="1")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--csv", default=None)
    ap.add_argument("--svg", default=None)
    ap.add_argument("--seed", type=int, default=42)
    ap.add_argument("--dtype", default="f64", choices=["f32", "f64"])
    ap.add_argument("--bounds", action="store_true",
                    help="append the HBM traffic-model columns alg_bytes, hbm_bound_s, "
                         "dram_bytes, dram_per_alg")
    ap.add_argument("--measure-dram", action="store_true",
                    help="with --bounds: measure dram_bytes with ncu (one extra pass per run)")
    ap.add_argument("--gpus", type=int, default=1,
                    help="shard every configuration over this many GPUs (cabl_mgpu C ABI)")
    ap.add_argument("--mgpu", action="store_true",
                    help="go through the multi-GPU C ABI even at --gpus 1")
    ap.add_argument("--dram-pass", action="store_true", help=argparse.SUPPRESS)
    raw = list(sys.argv[1:] if argv is None else argv)
    a = ap.parse_args(argv)
    try:
        if a.describe:
            from . import machine
            print(json.dumps(machine.descriptor_of(machine.describe_device(0),
                                                   4 if a.dtype == "f32" else 8), indent=2))
            return 0
        cfg = SweepConfig(bounds=a.bounds, kernels=list(KERNELS) if a.kernel == "all" else [a.kernel],
                          sizes=parse_sizes(a.sizes), rects=parse_rects(a.rect),
                          threads=[int(t) for t in a.threads.split(",") if t.strip()],
                          reps=a.reps, seed=a.seed, dtype=a.dtype, gpus=a.gpus)
        if a.machine:
            cfg.max_threads = load_descriptor(a.machine).cores
        if a.measure_dram and not a.bounds:
            raise ValueError("--measure-dram needs --bounds")
        if a.measure_dram and (a.gpus > 1 or a.mgpu):
            raise ValueError("--measure-dram profiles one GPU (ncu); drop --gpus / --mgpu")
        if a.dram_pass:  # internal: one marked call per configuration, no output
            _, failures = run_sweep(cfg, nvtx=True)
            return 0 if not failures else 1
        records, failures = run_sweep(cfg, use_mgpu=a.mgpu)
        if a.measure_dram and records:
            import tempfile
            keep = [t for t in raw if t not in ("--measure-dram",)]
            drop_next = {"--csv", "--svg"}
            argv2, skip = [], False
            for t in keep:
                if skip:
                    skip = False
                    continue
                if t in drop_next:
                    skip = True
                    continue
                if t.split("=")[0] in drop_next:
                    continue
                argv2.append(t)
            with tempfile.TemporaryDirectory() as td:
                measure_dram(argv2, records, Path(td))
        for f in failures:
            print("FAILED " + f, file=sys.stderr)
        if records:
            text = emit_csv(records)
            if a.csv:
                Path(a.csv).write_text(text)
            else:
                sys.stdout.write(text)
            if a.svg:
                Path(a.svg).write_text(emit_svg(records))
        return 0 if not failures else 1
    except Exception as e:  # noqa: BLE001
        print(f"error: {e}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
