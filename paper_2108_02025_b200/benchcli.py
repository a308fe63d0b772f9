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
shapes, CSV columns dtype, gbs, roofline_frac (of the measured HBM peak);
timing is CUDA events with the L2 flushed between repetitions; `threads` is
validated against the descriptor (as the reference does) and recorded, but
does not shape the GPU launch.  The spot check is an independent fp64
PyTorch computation on the device with the reference's tolerances (dot and
gemv: n*eps*sum|a_i b_i|; ger: one rounding of x_i*y_j + C_ij).
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
CSV_GPU_SUFFIX = ",dtype,gbs,roofline_frac"
# --bounds: the HBM traffic model in place of the reference's CPU-cache bound
# columns (reference bench.hpp:214-226, io_bounds.hpp report()): the bytes the
# operation must move and the time they take at the measured
# HBM peak — the B200 lower bound the measured median is compared against.
CSV_BOUNDS_SUFFIX = ",alg_bytes,hbm_bound_s"
KERNELS = ("dot", "ger", "gemv-row", "gemv-col")


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
    alg_bytes: int | None = None      # --bounds
    hbm_bound_s: float | None = None  # --bounds


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
             _g9(r.roofline_frac)]
        if bounds:
            f += [str(r.alg_bytes), _g9(r.hbm_bound_s)]
        lines.append(",".join(f))
    return "\n".join(lines) + "\n"


def parse_csv(text: str) -> list[BenchRecord]:
    rows = text.splitlines()
    if not rows:
        raise ValueError("parse_csv: empty document")
    head = rows[0]
    bounds = head == CSV_HEADER + CSV_GPU_SUFFIX + CSV_BOUNDS_SUFFIX
    gpu = bounds or head == CSV_HEADER + CSV_GPU_SUFFIX
    if not gpu and head != CSV_HEADER:
        raise ValueError("parse_csv: unexpected header")
    want = 14 if bounds else (12 if gpu else 9)
    out = []
    for line in rows[1:]:
        if not line:
            continue
        f = line.split(",")
        if len(f) != want:
            raise ValueError("parse_csv: bad field count")
        r = BenchRecord(f[0], int(f[1]), int(f[2]), int(f[3]), int(f[4]), float(f[5]),
                        float(f[6]), float(f[7]), float(f[8]))
        if gpu:
            r.dtype, r.gbs, r.roofline_frac = f[9], float(f[10]), float(f[11])
        if bounds:
            r.alg_bytes, r.hbm_bound_s = int(f[12]), float(f[13])
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
def _alg_bytes(kernel: str, m: int, n: int, s: int) -> int:
    if kernel == "dot":
        return 2 * n * s
    if kernel.startswith("gemv"):
        return m * n * s + n * s + 2 * m * s
    return 2 * m * n * s + m * s + n * s


def run_config(kernel: str, m: int, n: int, threads: int, cfg: SweepConfig, flush, peak: float,
               failures: list[str]) -> BenchRecord | None:
    import torch

    from . import cabl
    dt = torch.float32 if cfg.dtype == "f32" else torch.float64
    s = 4 if cfg.dtype == "f32" else 8
    eps = float(torch.finfo(dt).eps)
    dev = torch.device("cuda", torch.cuda.current_device())
    pol = cabl.ExecPolicy(cabl.derive_blocking_plan(cabl.default_machine(cfg.max_threads)), threads)
    salt = zlib.crc32(kernel.encode()) * 1000003 + m * 31 + n  # stable across processes
    fill = lambda k, st: cabl.fill_uniform(torch.empty(k, dtype=dt, device=dev), cfg.seed + salt, st)  # noqa: E731
    rec = BenchRecord(kernel, 0 if kernel == "dot" else m, n, threads, cfg.reps, dtype=cfg.dtype)
    fail = None
    if kernel == "dot":
        x, y = fill(n, 1), fill(n, 2)
        got = cabl.dot(x, y, 0.0, pol)
        p = x.double() * y.double()
        want, sumabs = float(p.sum()), float(p.abs().sum())
        if abs(got - want) > n * eps * sumabs + 4 * eps * abs(want):
            fail = f"abs diff = {abs(got - want):.3e}"
        rec.checksum = got
        call = lambda: cabl.dot_into(x, y, 0.0, out1, pol)  # noqa: E731
        out1 = torch.empty(1, dtype=dt, device=dev)
    elif kernel == "ger":
        x, y, C0 = fill(m, 1), fill(n, 2), fill(m * n, 5)
        Cm = cabl.DenseMatrix.wrap(C0.clone(), m, n, cabl.Layout.RowMajor)
        cabl.ger(x, y, Cm, pol)
        prod = x.double()[:, None] * y.double()[None, :]
        exact = C0.double().view(m, n) + prod
        got = Cm.data.double().view(m, n)
        tol = eps * (C0.double().view(m, n).abs() + prod.abs()) + torch.finfo(dt).tiny
        if not bool(((got - exact).abs() <= tol).all()):
            fail = "not within one rounding of x_i*y_j + C_ij"
        rec.checksum = float(Cm.data.double().sum())
        call = lambda: cabl.ger(x, y, Cm, pol)  # noqa: E731
    else:
        lay = cabl.Layout.RowMajor if kernel == "gemv-row" else cabl.Layout.ColMajor
        A, x, c0 = fill(m * n, 3), fill(n, 1), fill(m, 4)
        Am = cabl.DenseMatrix.wrap(A, m, n, lay)
        c = c0.clone()
        f = cabl.gemv_row_major if kernel == "gemv-row" else cabl.gemv_col_major
        f(Am, x, c, pol)
        A2 = A.double().view(m, n) if lay == cabl.Layout.RowMajor else A.double().view(n, m).t()
        want = c0.double() + A2 @ x.double()
        rowabs = A2.abs() @ x.double().abs()
        if not bool(((c.double() - want).abs() <= n * eps * rowabs + 4 * eps * want.abs()).all()):
            fail = f"max abs diff = {float((c.double() - want).abs().max()):.3e}"
        rec.checksum = float(c.double().sum())
        call = lambda: f(Am, x, c, pol)  # noqa: E731
    if fail:
        failures.append(f"kernel={kernel} m={rec.m} n={n} threads={threads}: oracle mismatch, {fail}")
        return None
    call()  # warm-up
    times = []
    for _ in range(cfg.reps):
        flush()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        call()
        b.record()
        torch.cuda.synchronize()
        times.append(a.elapsed_time(b) / 1e3)
    rec.min_s = min(times)
    rec.median_s = max(statistics.median(times), 1e-12)
    flops = 2 * n if kernel == "dot" else 2 * m * n
    rec.gflops = flops / rec.median_s / 1e9
    rec.gbs = _alg_bytes(kernel, m, n, s) / rec.median_s / 1e9
    rec.roofline_frac = rec.gbs / peak
    if cfg.bounds:
        rec.alg_bytes = _alg_bytes(kernel, m, n, s)
        rec.hbm_bound_s = rec.alg_bytes / (peak * 1e9)
    return rec


def run_sweep(cfg: SweepConfig) -> tuple[list[BenchRecord], list[str]]:
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
    if not torch.cuda.is_available():
        raise RuntimeError("no CUDA device (the B200 bench has no CPU path)")
    peak = _peak()
    wbuf = torch.empty(128 << 20, dtype=torch.float32, device="cuda")
    rbuf = torch.zeros(128 << 20, dtype=torch.float32, device="cuda")

    def flush():  # 512 MiB write then 512 MiB read: > L2, and no dirty lines left
        wbuf.zero_()
        rbuf.sum()

    records, failures = [], []
    for k in cfg.kernels:
        shapes = [(s, s) for s in cfg.sizes] + ([] if k == "dot" else list(cfg.rects))
        for m, n in shapes:
            for t in cfg.threads:
                r = run_config(k, m, n, t, cfg, flush, peak, failures)
                if r is not None:
                    records.append(r)
    return records, failures


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
                    help="append the HBM traffic-model columns alg_bytes, hbm_bound_s")
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
                          reps=a.reps, seed=a.seed, dtype=a.dtype)
        if a.machine:
            cfg.max_threads = load_descriptor(a.machine).cores
        records, failures = run_sweep(cfg)
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
