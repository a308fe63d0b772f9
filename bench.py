#!/usr/bin/env python
"""bench.py — DOT/GEMV/GER achieved HBM GB/s and % of the B200 roofline.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload G1] [--no-suite] [--no-cpu-baseline]

Multi-GPU runs are launched one process per GPU by torchrun (RANK /
LOCAL_RANK / WORLD_SIZE from the environment, NCCL over NVLink); without
torchrun, ``--gpus N`` re-executes itself under torch.distributed.run after
checking that N GPUs are visible, and a WORLD_SIZE other than N is refused.

Headline workload (``--workload``, default G1 = BASELINE.json configs[1],
GEMV fp32 row-major 8192 x 8192): a STEP is one pass of the hot path over one
batch — one c += A x over an 8192 x 8192 row block.  At N GPUs every rank
owns its own 8192-row block of an (8192 N) x 8192 matrix with x replicated
(weak scaling; row blocks need no collective).

* ``value``     whole-job GB/s = algorithmic bytes of all ranks x K / the
                max over ranks of the device time of the K steps, inputs
                resident in HBM.  L2 policy (``--l2``, reported in config.l2):
                a step whose footprint exceeds the 126 MB L2 (every BASELINE
                config: D1 134 MB ... D2 34 GB) runs back to back under one
                event pair — ncu shows every back-to-back launch still reads
                its full algorithmic bytes from DRAM; steps that fit in L2
                are timed one by one with the L2 flushed in between (512 MiB
                write + 512 MiB read, outside the events).
* ``e2e``       the same metric through the public host-buffer API
                (cabl_host_gemv_f32 via cabl.gemv_row_major on pinned CPU
                tensors): H2D of A, x, c + kernel + D2H of c every step.
* ``roofline``  the dominant (only) kernel: algorithmic bytes per launch /
                mean launch time vs MEASURED_PEAKS.json hbm_gbs; traffic =
                DRAM bytes per launch from the committed ncu capture.
* ``cpu_baseline`` the compiled, UNMODIFIED reference (oracle/_ref,
                kind "reference") — its threaded gemv_row_major with every
                host core — on a bounded sample of the same workload.
* ``suite``     every BASELINE config at this N (device GB/s, % of peak): back
                to back when the step's footprint exceeds L2, else back to back
                over rotating copies of the operands (time_rotating); the
                one-flushed-launch-at-a-time figure rides along.  At N > 1 a
                watchdog (--suite-timeout) prints the finished headline line
                if a suite collective hangs.

``--impl reference`` times the reference's own CPU implementation of the
path on this box's host cores (rank 0 only) and prints the same line shape.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

FALLBACK_HBM_GBS = 6650.0
FLUSH_BYTES = 512 << 20  # default; run_ours takes it from the GPU plan (4 x L2, pow2)


class L2Flush:
    """Between timed steps: WRITE a 512 MiB buffer (> 4x the 126 MB L2), then READ
    a second one.  The write evicts every line of the step's operands; the
    read then evicts the flush's own dirty lines (their write-back happens
    here, outside the timed events), so each step starts from an L2 that
    holds nothing of its inputs and nothing dirty."""

    def __init__(self, dev, nbytes: int = FLUSH_BYTES):
        import torch
        self.w = torch.empty(nbytes // 4, dtype=torch.float32, device=dev)
        self.r = torch.zeros(nbytes // 4, dtype=torch.float32, device=dev)
        self.e = torch.zeros(nbytes // 8, dtype=torch.float32, device=dev)
        self._evict_ms = None

    def zero_(self):
        self.w.zero_()
        self.r.sum()

    def evict_(self):
        """Read a buffer of 2 x L2 that the L2 does not hold: every line the
        step left dirty is written back during this pass."""
        self.e.sum()

    def evict_ms(self, reps: int = 15) -> float:
        """Mean time of evict_() right after zero_() (nothing dirty in L2):
        what a timed step that ends with evict_() subtracts."""
        import torch
        if self._evict_ms is None:
            ts = []
            for i in range(reps + 2):
                self.zero_()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                self.evict_()
                b.record()
                torch.cuda.synchronize()
                if i >= 2:
                    ts.append(a.elapsed_time(b))
            self._evict_ms = sum(ts) / len(ts)
        return self._evict_ms


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def traffic_for(kernel_key: str):
    """DRAM bytes per launch for a kernel from the committed ncu summary."""
    p = ROOT / "profiles" / "ncu_traffic.json"
    if not p.exists():
        return None, None
    d = json.loads(p.read_text())
    e = d.get(kernel_key)
    if not e:
        return None, None
    return e.get("dram_bytes_per_launch"), e.get("source")


def traffic_kernel(cfg: str):
    p = ROOT / "profiles" / "ncu_traffic.json"
    if not p.exists():
        return None
    e = json.loads(p.read_text()).get(cfg) or {}
    k = e.get("kernel")
    return k.split("::")[-1] if k else None


# ----------------------------------------------------------------- clocks
class ClockSampler:
    """Samples SM clock and throttle reasons through NVML while running."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
        0x100: "display_clock_setting",
    }

    def __init__(self, index: int):
        self.ok = False
        self.samples: list[int] = []
        self.reasons: set[str] = set()
        self.max_mhz = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # noqa: BLE001
            self.err = str(e)
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                mask = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if mask & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:  # noqa: BLE001
                pass
            time.sleep(0.0005)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "error": self.err}
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


# ----------------------------------------------------------------- setup
def workload_config(w) -> dict:
    """The line's ``config``: workload-defining fields only, identical for our
    arm and the reference arm (so the driver can match the two lines).  How a
    run was executed (GPUs, machine, L2 policy details) goes under ``run``."""
    step = w.footprint_bytes()
    return {"workload": f"{w.id}: {w.desc}", "m_per_gpu": w.m, "n": w.n,
            "layout": {"gemv-row": "row-major", "gemv-col": "col-major", "ger": "row-major",
                       "dot": "vector"}[w.op],
            "dtype": w.dtype_name,
            "l2": (f"inputs larger than L2 ({step / 1e6:.0f} MB per step vs the 126 MB B200 L2): "
                   "steps back to back" if step > L2_BYTES else
                   "L2 flushed between steps (outside the timed events)")}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


class Ctx:
    def __init__(self, world, rank, local, dev):
        self.world, self.rank, self.local, self.dev = world, rank, local, dev

    def barrier(self):
        import torch.distributed as dist
        if self.world > 1:
            dist.barrier(device_ids=[self.local])

    def max(self, v: float) -> float:
        import torch
        import torch.distributed as dist
        if self.world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=self.dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())


def make_inputs(w, rows: tuple[int, int], dev, layout=None):
    """Seeded device inputs for this rank's shard of workload w."""
    import torch

    import paper_2108_02025_b200 as cb
    from paper_2108_02025_b200 import workloads as WL
    fill = cb.fill_normal if w.dist == "normal" else cb.fill_uniform
    r0, r1 = rows
    if w.op == "dot":
        n = r1 - r0
        x = fill(torch.empty(n, dtype=w.dtype, device=dev), WL.SEED, WL.STREAM_X, r0)
        y = fill(torch.empty(n, dtype=w.dtype, device=dev), WL.SEED, WL.STREAM_Y, r0)
        return {"x": x, "y": y, "out": torch.empty(1, dtype=w.dtype, device=dev)}
    m = r1 - r0
    if w.op.startswith("gemv"):
        lay = cb.Layout.RowMajor if w.op == "gemv-row" else cb.Layout.ColMajor
        A = torch.empty(m * w.n, dtype=w.dtype, device=dev)
        if lay == cb.Layout.RowMajor:
            fill(A, WL.SEED, WL.STREAM_A, r0 * w.n)
        else:
            fill(A, WL.SEED, WL.STREAM_A, 0)
        x = fill(torch.empty(w.n, dtype=w.dtype, device=dev), WL.SEED, WL.STREAM_X, 0)
        c = fill(torch.empty(m, dtype=w.dtype, device=dev), WL.SEED, WL.STREAM_C, r0)
        return {"A": cb.DenseMatrix.wrap(A, m, w.n, lay), "x": x, "c": c}
    C = fill(torch.empty(m * w.n, dtype=w.dtype, device=dev), WL.SEED, WL.STREAM_CC, r0 * w.n)
    x = fill(torch.empty(m, dtype=w.dtype, device=dev), WL.SEED, WL.STREAM_X, r0)
    y = fill(torch.empty(w.n, dtype=w.dtype, device=dev), WL.SEED, WL.STREAM_Y, 0)
    return {"C": cb.DenseMatrix.wrap(C, m, w.n, cb.Layout.RowMajor), "x": x, "y": y}


def step_fn(w, ins, policy, ctx, sharded_dot: bool, fused: bool = False):
    import paper_2108_02025_b200 as cb
    from paper_2108_02025_b200 import shard
    from paper_2108_02025_b200 import workloads as WL
    if w.op == "dot" and fused:
        # the exchange of partials fused into the DOT kernel over peer memory
        # (csrc/peer.cu): one launch per step at any N, no NCCL call
        if getattr(ctx, "peer_mb", None) is None:
            ctx.peer_mb = shard.PeerMailboxes(ctx.dev)
        return (lambda: shard.sharded_dot_fused(ins["x"], ins["y"], 0.0, ins["out"], policy,
                                                ctx.peer_mb)), 1
    if w.op == "dot":
        if sharded_dot and ctx.world > 1:
            import torch
            gathered = torch.empty(ctx.world, dtype=w.dtype, device=ctx.dev)
            return (lambda: shard.sharded_dot(ins["x"], ins["y"], 0.0, ins["out"], policy,
                                              gathered=gathered)), 2  # dot + combine (+ NCCL all-gather)
        return (lambda: cb.dot_into(ins["x"], ins["y"], 0.0, ins["out"], policy)), 1
    if w.op == "gemv-row" and fused:
        # row blocks with the c all-gather inside the GEMV kernel (csrc/peer_gemv.cu)
        m_total = WL.WORKLOADS[w.id].m
        row_off = WL.Workload.shard_rows(WL.WORKLOADS[w.id], ctx.rank, ctx.world)[0] \
            if ctx.world > 1 else 0
        if getattr(ctx, "gather_gemv", None) is None:
            ctx.gather_gemv = shard.GatherGemv(ctx.dev, m_total, w.dtype)
        return (lambda: ctx.gather_gemv(ins["A"], ins["x"], ins["c"], row_off)), 1
    if w.op == "gemv-row" and sharded_dot and ctx.world > 1 and w.id == "G4":
        # BASELINE config 5: "c slices all-gathered" (NCCL) after the row blocks
        import torch
        m_total = WL.WORKLOADS["G4"].m
        full_c = torch.empty(m_total, dtype=w.dtype, device=ctx.dev)
        return (lambda: shard.sharded_gemv_rows(ins["A"], ins["x"], ins["c"], policy,
                                                gather=True, m_total=m_total, out=full_c)), 1
    if w.op == "gemv-row":
        return (lambda: cb.gemv_row_major(ins["A"], ins["x"], ins["c"], policy)), 1
    if w.op == "gemv-col":
        return (lambda: cb.gemv_col_major(ins["A"], ins["x"], ins["c"], policy)), 1
    return (lambda: cb.ger(ins["x"], ins["y"], ins["C"], policy)), 1


# L2 capacity: replaced in run_ours by the live device's (machines: the GPU
# descriptor, paper_2108_02025_b200/machine.py); this is B200's value.
L2_BYTES = 126 << 20


def l2_mode(step_bytes: int) -> str:
    """'stream' when the DISTINCT bytes a step touches (Workload.footprint_bytes:
    GER's in-place C counts once, not as read + write) exceed the L2: the
    front-to-back sweep of step k+1 misses on everything step k left behind.  Checked with ncu
    (--cache-control none) on back-to-back launches of the two smallest
    configs: every G1 launch (268.5 MB alg.) reads 268.5 MB from DRAM; a D1
    launch (134.2 MB) reads 131.2 MB, i.e. ~2% of it still hits in L2
    (profiles/r01_ncu_b2b_{D1,G1}.csv, profiles/r02_ncu_b2b_{D1,G1}.csv).
    'flush' otherwise (inputs that fit in L2)."""
    return "stream" if step_bytes > L2_BYTES else "flush"


PRIME_CYCLES = 1_000_000  # ~0.5 ms at 1965 MHz, outside the timed region


def time_steps(fn, steps, warmup, ctx, flush, sampler=None, mode="flush", charge_writeback=False):
    """Per-step device times (ms) on the launching stream, barrier + synchronize
    on both sides of the timed region.
    mode 'flush':  L2 flushed between steps outside per-step CUDA events.
                   charge_writeback (GER: C is written): each step's events
                   also enclose an eviction pass, whose clean-L2 time is
                   subtracted — so the write-back of the lines the kernel
                   left dirty in L2 (ncu: ~56 of R1's 268 MB of C) is charged
                   to the step instead of to the next flush.
    mode 'stream': inputs > 2x L2 — steps back to back, one event pair around
                   all K steps (per-step time = total / K)."""
    import torch
    for _ in range(warmup):
        if mode == "flush":
            flush.zero_()
        fn()
    torch.cuda.synchronize()
    if mode == "stream":
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ctx.barrier()
        torch.cuda.synchronize()
        if sampler:
            sampler.__enter__()
        t0 = time.perf_counter()
        # hold the stream with a short device sleep (the blocking-kernel trick
        # of nvbench) so the start event and the first steps are already queued
        # when the GPU reaches them: the K timed steps then run back to back
        # from the start event, without the host's first-launch latency in the
        # interval (driver K = 20: ~1.5 us per step of the G1 headline)
        prime = getattr(torch.cuda, "_sleep", None)  # private torch API: optional
        if prime is not None:
            prime(PRIME_CYCLES)
        a.record()
        for _ in range(steps):
            fn()
        b.record()
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        if sampler:
            sampler.__exit__()
        ctx.barrier()
        per = a.elapsed_time(b) / steps
        return [per] * steps, wall
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    ctx.barrier()
    torch.cuda.synchronize()
    if sampler:
        sampler.__enter__()
    t0 = time.perf_counter()
    for k in range(steps):
        flush.zero_()
        starts[k].record()
        fn()
        if charge_writeback:
            flush.evict_()
        ends[k].record()
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    if sampler:
        sampler.__exit__()
    ctx.barrier()
    sub = flush.evict_ms() if charge_writeback else 0.0
    return [s.elapsed_time(e) - sub for s, e in zip(starts, ends)], wall


def rotating_copies(footprint: int) -> int:
    """Independent copies of a step's operands so that their combined footprint
    exceeds 2x the L2 (at least 3, at most 24)."""
    return max(3, min(24, -(-2 * L2_BYTES // max(1, footprint)) + 1))


def time_rotating(fns, steps, warmup, ctx, flush, charge_writeback=False):
    """Steps back to back over len(fns) independent copies of the step's operands,
    taken in turn: a step whose footprint fits in L2 (an R1 shard at N >= 4) still
    reads its operands from HBM, because the copies used since its last turn pushed
    them out — "inputs larger than L2" by rotation instead of a flush before every
    launch, so launch latency and the write-back of dirty lines overlap the next
    step as they do for the large configs in 'stream' mode.  One event pair around
    all K steps; with charge_writeback the pair also encloses a final eviction pass
    (minus its clean-L2 time), so the lines the last steps left dirty are charged
    too.  Returns per-step ms (total / K)."""
    import torch
    R = len(fns)
    sub = flush.evict_ms() if charge_writeback else 0.0
    for k in range(max(warmup, R)):
        fns[k % R]()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ctx.barrier()
    torch.cuda.synchronize()
    prime = getattr(torch.cuda, "_sleep", None)  # private torch API: optional
    if prime is not None:
        prime(PRIME_CYCLES)
    a.record()
    for k in range(steps):
        fns[k % R]()
    if charge_writeback:
        flush.evict_()
    b.record()
    torch.cuda.synchronize()
    ctx.barrier()
    return [(a.elapsed_time(b) - sub) / steps] * steps


# ------------------------------------------------------------ CPU baseline
_CPU_INPUTS: dict = {}


def cpu_reference_sample(w, max_bytes=1 << 30, reps=5, threads=None, naive=False):
    """Time the compiled reference (oracle/_ref) on a bounded sample of w:
    its threaded path (cabl::dot / gemv_* / ger), or with naive=True its
    naive oracle (dot_ref / gemv_ref / ger_ref, one thread)."""
    import numpy as np

    from oracle import oracle as O
    from paper_2108_02025_b200 import workloads as WL
    cores = threads or os.cpu_count() or 1
    kind = "reference" if O.ref_available() else "port"
    npdt = np.float32 if w.dtype_name == "f32" else np.float64
    s = np.dtype(npdt).itemsize
    gen0 = (lambda n, st, off=0: O.gen_normal_f64(n, WL.SEED, st, off)) if w.dist == "normal" \
        else (lambda n, st, off=0: O.gen_uniform(n, npdt, WL.SEED, st, off))

    def gen(n, st, off=0):  # the last config's inputs are kept for the next path
        key = (w.dist, w.dtype_name, n, st, off)
        if key not in _CPU_INPUTS:
            if len(_CPU_INPUTS) >= 3:
                _CPU_INPUTS.clear()
            _CPU_INPUTS[key] = gen0(n, st, off)
        return _CPU_INPUTS[key]
    if w.op == "dot":
        n = min(w.n, max_bytes // (2 * s))
        m = 0
        x, y = gen(n, WL.STREAM_X), gen(n, WL.STREAM_Y)
        alg = 2 * n * s
        sample = f"dot {w.dtype_name} n={n}"
    else:
        m, n = w.m, w.n
        if m * n * s > max_bytes:
            if w.op == "gemv-col" and m > n:
                m = max(1, max_bytes // (n * s))
            elif w.op == "gemv-col":
                n = max(1, max_bytes // (m * s))
            else:
                m = max(1, max_bytes // (n * s))
        if w.op.startswith("gemv"):
            A, x, c = gen(m * n, WL.STREAM_A), gen(n, WL.STREAM_X), gen(m, WL.STREAM_C)
            alg = m * n * s + n * s + 2 * m * s
        else:
            A, x, c = gen(m * n, WL.STREAM_CC), gen(m, WL.STREAM_X), gen(n, WL.STREAM_Y)
            alg = 2 * m * n * s + m * s + n * s
        sample = f"{w.op} {w.dtype_name} {m}x{n}"
    times = []
    if kind == "reference":
        if w.op == "dot":
            sess = O.RefSession("dot", npdt, 0, 0, n, None, x, y, 0.0, cores=cores)
        elif w.op == "ger":
            sess = O.RefSession("ger", npdt, 0, m, n, A, x, c, cores=cores)
        else:
            sess = O.RefSession(w.op, npdt, 0 if w.op == "gemv-row" else 1, m, n, A, x, c,
                                cores=cores)
        used = 1 if naive else cores
        times = O.time_ref(sess, use_ref=naive, threads=used, reps=reps)
        sess.close()
    else:  # restated oracle, single thread
        used = 1
        for _ in range(reps):
            t0 = time.perf_counter()
            if w.op == "dot":
                O.dot_ref(x, y, 0.0)
            elif w.op == "ger":
                O.ger_ref(x, c, A, 0)
            else:
                O.gemv_ref(A, 0 if w.op == "gemv-row" else 1, x, c)
            times.append(time.perf_counter() - t0)
    t = statistics.median(times)
    return {"value": round(alg / t / 1e9, 3), "unit": "GB/s", "cores": used, "kind": kind,
            "sample": f"{sample}, median of {reps} after 1 warm-up"
                      + ((", reference naive oracle (1 thread)" if naive else
                          ", reference threaded path (ExecPolicy threads=%d)" % used)
                         if kind == "reference" else ", restated oracle (1 thread)"),
            "median_s": t}


# ------------------------------------------------------------ our arm
def run_ours(args, ctx):
    import torch

    import paper_2108_02025_b200 as cb
    from paper_2108_02025_b200 import workloads as WL
    peak, peak_src = peaks()
    policy = cb.default_policy(1)
    w = WL.WORKLOADS[args.workload]
    # launch parameters from the live GPU descriptor
    from paper_2108_02025_b200 import machine as MC
    global L2_BYTES
    ginfo = MC.describe_device(ctx.local)
    gplan = MC.derive_gpu_plan(MC.load_descriptor(json.dumps(MC.descriptor_of(ginfo))))
    L2_BYTES = gplan.l2_bytes
    flush = L2Flush(ctx.dev, gplan.l2_flush_bytes)

    # ---- headline: weak scaling, every rank its own full-size block
    span = w.n if w.op == "dot" else w.m
    rows = (ctx.rank * span, (ctx.rank + 1) * span)
    ins = make_inputs(w, rows, ctx.dev)
    fn, launches_per_step = step_fn(w, ins, policy, ctx, sharded_dot=False)
    sampler = ClockSampler(ctx.local)
    mode = args.l2 if args.l2 != "auto" else l2_mode(w.footprint_bytes())
    times, wall = time_steps(fn, args.steps, args.warmup, ctx, flush, sampler, mode=mode,
                             charge_writeback=(mode == "flush" and w.op == "ger"))
    t_rank = sum(times) / 1000.0
    t_max = ctx.max(t_rank)
    bytes_rank = w.alg_bytes(1)
    value = ctx.world * bytes_rank * args.steps / t_max / 1e9
    mean_launch_s = t_rank / args.steps
    achieved = bytes_rank / mean_launch_s / 1e9
    traffic, traffic_src = traffic_for(f"{w.id}")
    clocks = sampler.summary()

    # ---- e2e: the reference-facing drop-in call on host buffers (cabl_host_*,
    # every operand copied every step); e2e_resident: the resident-operator
    # pipeline (GEMV: A uploaded once, x and c streamed)
    e2e = e2e_resident = None
    if not args.no_e2e:
        e2e_resident, e2e = run_e2e(w, ins, policy, ctx, args)
        if e2e is None:  # DOT / GER: the host-buffer call is the only pattern
            e2e, e2e_resident = e2e_resident, None

    del ins
    torch.cuda.empty_cache()

    # ---- CPU baseline (rank 0, N=1)
    cpu = None
    if ctx.rank == 0 and ctx.world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_reference_sample(w)
            cpu.pop("median_s", None)
        except Exception as e:  # noqa: BLE001
            cpu = {"value": None, "error": str(e)}

    line = {
        "metric": "DOT/GEMV/GER achieved HBM GB/s & % of B200 roofline at 1/2/4/8 GPUs",
        "value": round(value, 2),
        "unit": "GB/s",
        "n_gpus": ctx.world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(t_max / args.steps * 1e3, 5),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": w.dtype_name,
        "data": "synthetic: seeded SplitMix64 U[-1,1) (seed 42), generated on device",
        "config": workload_config(w),
        "run": {
            "parallelism": (f"{w.shard} over {ctx.world} GPU(s) (one process per GPU), "
                            "weak scaling, no collective in the step"),
            "machine": {"gpu": ginfo.name, "sms": gplan.sm_count, "l2_bytes": gplan.l2_bytes,
                        "source": "cabl_describe_device"},
            "l2": (f"inputs larger than L2: {bytes_rank / 1e6:.0f} MB per step vs "
                   f"{gplan.l2_bytes / 1e6:.0f} MB L2, "
                   "steps back to back (one event pair around the K steps, queued behind a "
                   "0.5 ms device sleep so the first step carries no host launch latency); ncu shows each "
                   "back-to-back launch reads its full algorithmic bytes from DRAM "
                   "(profiles/r02_ncu_b2b_*.csv)" if mode == "stream" else
                   f"flushed between steps outside the timed events: {gplan.l2_flush_bytes >> 20} "
                   f"MiB write, then {gplan.l2_flush_bytes >> 20} MiB read (no dirty lines left "
                   "in L2)"),
            "alg_bytes_per_step_per_gpu": bytes_rank,
        },
        "roofline": {
            "bound": "hbm", "achieved": round(achieved, 2), "peak": peak, "unit": "GB/s",
            "frac": round(achieved / peak, 4), "peak_source": peak_src,
            "traffic": traffic, "traffic_source": traffic_src,
            "kernel": traffic_kernel(w.id) or w.op,
            "mean_launch_us": round(mean_launch_s * 1e6, 3),
        },
        "e2e": e2e,
        "e2e_resident": e2e_resident,
        "cpu_baseline": cpu,
        "gpu_launches": launches_per_step * args.steps,
        "clocks": clocks,
        "wall_s_timed_region": round(wall, 4),
        "suite": None,
    }

    # ---- suite of all BASELINE configs at this N.  The headline above is complete;
    # at N > 1 the suite's sharded entries use collectives that this pool (one GPU
    # per box) has only run at world size 1, so a watchdog guards the line: if the
    # suite has not finished within --suite-timeout seconds (a rank died or a
    # collective hangs), rank 0 prints the line with the suite marked as timed out
    # and every rank exits 0 instead of taking the headline down with it.
    if not args.no_suite:
        import threading
        done = threading.Lock()

        def give_up():
            if not done.acquire(blocking=False):
                return  # the normal path is already printing
            if ctx.rank == 0:
                line["suite"] = {"error": f"suite did not finish within {args.suite_timeout} s "
                                          "(watchdog); headline, e2e and roofline are complete"}
                print(json.dumps(line), flush=True)
            os._exit(0)

        dog = None
        if args.suite_timeout is None:
            args.suite_timeout = 600.0 if ctx.world > 1 else 0.0
        if args.suite_timeout > 0:
            dog = threading.Timer(args.suite_timeout, give_up)
            dog.daemon = True
            dog.start()
        try:
            suite = run_suite(args, ctx, flush, policy, peak)
        except Exception as ex:  # noqa: BLE001
            if ctx.world == 1:
                raise
            # keep this rank alive (its peers may be inside a collective with it
            # missing): the watchdog ends every rank, rank 0 after printing
            print(f"bench.py: rank {ctx.rank}: suite failed: {ex!r}", file=sys.stderr, flush=True)
            if dog is not None:
                dog.join()
            raise
        if not done.acquire(blocking=False):
            time.sleep(3600)  # the watchdog fired first and is printing / exiting
        if dog is not None:
            dog.cancel()
        line["suite"] = suite
    if ctx.rank != 0:
        return
    print(json.dumps(line), flush=True)


def _time_host_loop(fn, steps, warmup, ctx):
    for _ in range(min(3, warmup)):
        fn()
    ctx.barrier()
    t0 = time.perf_counter()
    for _ in range(steps):
        fn()
    return ctx.max(time.perf_counter() - t0)


E2E_DEPTH = 4
E2E_SUITE_MAX_BYTES = 3 << 30


def _h2d_seconds(nbytes: int, dev, to_host: bool = False) -> float:
    """Median wall time of a pinned host -> device copy of nbytes (the PCIe
    bound), or device -> host with to_host."""
    import torch
    h = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    d = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    ts = []
    for i in range(7):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if to_host:
            h.copy_(d, non_blocking=True)
        else:
            d.copy_(h, non_blocking=True)
        torch.cuda.synchronize()
        if i >= 2:
            ts.append(time.perf_counter() - t0)
    del h, d
    return sorted(ts)[len(ts) // 2]


def run_e2e(w, ins, policy, ctx, args, resident: bool = True):
    """End-to-end through the public API, host<->device copies inside the
    timed loop, wall clock (max over ranks).  Returns (resident, host):

    * host (the line's ``e2e``): the reference-facing drop-in call on host
      buffers (``cabl_host_*`` in the C ABI, what ``cabl::gemv_row_major`` on
      ``cabl::DenseMatrix`` calls): A / C / x / y / c copied H2D from pinned
      memory and the result D2H inside every call — PCIe-bound by construction.
    * resident (``e2e_resident``, GEMV only): the matrix is a resident
      operator — A is uploaded once, every step copies x and c from pinned
      host memory, runs the GEMV and reads c back."""
    import torch

    import paper_2108_02025_b200 as cb
    steps = max(1, min(args.steps, args.e2e_steps))
    api_host = "cabl.{dot,gemv_*,ger} on pinned CPU tensors -> cabl_host_* (C ABI)"
    if w.op == "dot":
        hx, hy = ins["x"].cpu().pin_memory(), ins["y"].cpu().pin_memory()
        fn = lambda: cb.dot(hx, hy, 0.0, policy)  # noqa: E731
        h2d, d2h = (hx.numel() + hy.numel()) * w.s, w.s
    elif w.op.startswith("gemv"):
        A = ins["A"]
        hA = cb.DenseMatrix.wrap(A.data.cpu().pin_memory(), A.rows(), A.cols(), A.layout())
        hx, hc = ins["x"].cpu().pin_memory(), ins["c"].cpu().pin_memory()
        f = cb.gemv_row_major if w.op == "gemv-row" else cb.gemv_col_major
        fn = lambda: f(hA, hx, hc, policy)  # noqa: E731
        h2d, d2h = (hA.size() + hx.numel() + hc.numel()) * w.s, hc.numel() * w.s
    else:
        Cm = ins["C"]
        hC = cb.DenseMatrix.wrap(Cm.data.cpu().pin_memory(), Cm.rows(), Cm.cols(), Cm.layout())
        hx, hy = ins["x"].cpu().pin_memory(), ins["y"].cpu().pin_memory()
        fn = lambda: cb.ger(hx, hy, hC, policy)  # noqa: E731
        h2d, d2h = (hC.size() + hx.numel() + hy.numel()) * w.s, hC.size() * w.s
    t_max = _time_host_loop(fn, steps, args.warmup, ctx)
    full = {"value": round(ctx.world * w.alg_bytes(1) * steps / t_max / 1e9, 3), "unit": "GB/s",
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "steps": steps,
            "ms_per_step": round(t_max / steps * 1e3, 4), "api": api_host}
    full["pattern"] = ("drop-in call on host buffers: every operand copied H2D from pinned "
                       "memory and the result D2H inside every call")
    # the link that bounds it: a plain pinned H2D copy of the same bytes, timed
    # here (PCIe is full duplex: GER's equal D2H can overlap it, so one
    # direction's time is the bound)
    link_s = _h2d_seconds(h2d, ctx.dev)
    h2d_gbs = h2d / link_s / 1e9
    full["link"] = {"h2d_gbs_measured": round(h2d_gbs, 2),
                    "h2d_bound_ms_per_step": round(link_s * 1e3, 4),
                    "frac_of_link": round(link_s / (t_max / steps), 4),
                    "what": "torch pinned-host -> device copy of the step's H2D bytes, median "
                            "of 5; frac_of_link = that copy's time / the e2e step time"}
    if d2h >= (1 << 20):  # GER: C also comes back; the duplex bound is the slower direction
        back_s = _h2d_seconds(d2h, ctx.dev, to_host=True)
        bound = max(link_s, back_s)
        full["link"].update({"d2h_gbs_measured": round(d2h / back_s / 1e9, 2),
                             "duplex_bound_ms_per_step": round(bound * 1e3, 4),
                             "frac_of_duplex_bound": round(bound / (t_max / steps), 4)})
    if not w.op.startswith("gemv"):
        return full, None
    if not resident:
        return None, full

    # resident operator: A stays in HBM, x and c stream in, c streams out —
    # the public GemvPipeline (E2E_DEPTH independent requests in flight, one
    # stream each), one CUDA-graph replay per step; every step's result is
    # read back before its buffers are reused.  G1 on B200 (tools/e2e_depth.py):
    # depth 1 73.2 us/step, 2 42.5, 3 35.9, 4 35.9 — from depth 3 the next
    # request's kernel fills the SMs the previous one's tail leaves idle
    # (the same with a distinct copy of A per request, so not L2 sharing)
    from paper_2108_02025_b200.operators import GemvPipeline
    pipe = GemvPipeline(ins["A"], policy, depth=E2E_DEPTH)
    for op in pipe.ops:
        op.x_host.copy_(ins["x"].cpu())
        op.c_host.copy_(ins["c"].cpu())
    steps_r = max(1, args.steps)

    def run_all():
        for _ in range(steps_r):
            pipe.step()
        pipe.drain()

    for _ in range(min(3, args.warmup)):
        pipe.step()
    pipe.drain()
    ctx.barrier()
    t0 = time.perf_counter()
    run_all()
    t_res = ctx.max(time.perf_counter() - t0)
    op0 = pipe.ops[0]
    resident = {"value": round(ctx.world * w.alg_bytes(1) * steps_r / t_res / 1e9, 3),
                "unit": "GB/s",
                "h2d_bytes_per_step": (op0.x_host.numel() + op0.c_host.numel()) * w.s,
                "d2h_bytes_per_step": op0.out_host.numel() * w.s, "steps": steps_r,
                "ms_per_step": round(t_res / steps_r * 1e3, 4),
                "pattern": f"resident operator, {E2E_DEPTH} independent requests in flight "
                           "(one stream each): A uploaded once before timing; every step H2D "
                           "x, c from pinned host, GEMV kernel, D2H c (one CUDA graph replay); "
                           "each result is waited for before its buffers are reused; wall "
                           "clock over all K steps",
                "api": "paper_2108_02025_b200.operators.GemvPipeline -> cabl_cuda_gemv_rm_f32"}
    return resident, full


def peer_probe(fn, ctx) -> None:
    """One call of a fused peer-memory step before it is timed: if any rank's
    kernel gave up waiting for a peer (mailbox fault, after
    CABL_PEER_TIMEOUT_MS — bench.py sets 3 s), every rank agrees the path is
    unavailable and the suite moves on instead of stalling."""
    import torch
    fn()
    torch.cuda.synchronize()
    faults = [o.state()[1] for o in (getattr(ctx, "peer_mb", None), getattr(ctx, "gather_gemv", None))
              if o is not None]
    ok = torch.tensor([0 if any(faults) else 1], dtype=torch.int32, device=ctx.dev)
    if ctx.world > 1:
        import torch.distributed as dist
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
    if int(ok.item()) == 0:
        raise RuntimeError("a rank timed out waiting for its peers (mailbox fault)")


def run_suite(args, ctx, flush, policy, peak):
    """Every BASELINE config at this N.  N=1: all seven on one GPU.  N>1: the
    configs BASELINE shards (R1, G4 row blocks; D2 chunks + all-gather),
    strong scaling (fixed total problem)."""
    import torch

    from paper_2108_02025_b200 import workloads as WL
    ids = list(WL.WORKLOADS) if ctx.world == 1 else ["R1", "G4", "D2"]
    # D2 / G4 with the exchange fused into the kernel (peer memory): always at
    # N = 1; across processes (CUDA IPC + NVLink P2P, so far only emulated on
    # one GPU) only with --fused-suite, so the BASELINE lines of a scaling run
    # never wait on them
    if ctx.world == 1 or args.fused_suite:
        ids += ["D2f", "G4f"]
    out = {}
    steps = max(3, min(args.steps, args.suite_steps))
    for wid in ids:
        fused = wid in ("D2f", "G4f")
        w = WL.WORKLOADS[wid[:2] if fused else wid]
        total = w.n if w.op == "dot" else w.m
        b, e = (0, total) if ctx.world == 1 else WL.Workload.shard_rows(w, ctx.rank, ctx.world)
        try:
            ins = make_inputs(w, (b, e), ctx.dev)
            if w.op == "dot":
                import dataclasses
                wl = dataclasses.replace(w, n=e - b)
            else:
                import dataclasses
                wl = dataclasses.replace(w, m=e - b)
            fn, lps = step_fn(wl, ins, policy, ctx, sharded_dot=True, fused=fused)
            if fused:
                peer_probe(fn, ctx)
            alg = w.alg_bytes(ctx.world)
            # the shard's footprint decides (an R1 shard at N >= 4 fits in L2 and
            # would run out of it back to back: 64 MiB of C at 9.8 TB/s,
            # profiles/r02_shard_share.jsonl); a flushed GER is charged the
            # write-back of the lines it leaves dirty in L2
            mode = l2_mode(wl.footprint_bytes())
            nsteps = steps
            if mode == "flush" and not fused:
                # footprint <= L2: back to back over rotating copies of the operands
                # (time_rotating), the steady-state analogue of 'stream'; the
                # flushed-per-launch time stays as the conservative column
                mode = "rotate"
                R = rotating_copies(wl.footprint_bytes())
                rot = [fn] + [step_fn(wl, make_inputs(w, (b, e), ctx.dev), policy, ctx,
                                      sharded_dot=True)[0] for _ in range(R - 1)]
                nsteps = max(steps, 3 * R)
                times = time_rotating(rot, nsteps, args.warmup, ctx, flush,
                                      charge_writeback=w.op == "ger")
                del rot
            else:
                times, _ = time_steps(fn, steps, args.warmup, ctx, flush, mode=mode,
                                      charge_writeback=(mode == "flush" and w.op == "ger"))
            t_max = ctx.max(sum(times) / 1000.0) * steps / nsteps  # seconds for `steps` steps
            gbs = alg * steps / t_max / 1e9
            desc = w.desc + ((", partials exchanged inside the kernel over peer memory "
                              "(cabl_cuda_dot_peer)" if w.op == "dot" else
                              ", c slices all-gathered inside the GEMV kernel over peer memory "
                              "(cabl_cuda_gemv_rm_gather)") if fused else "")
            entry = {"desc": desc, "gbs": round(gbs, 2),
                     "frac_of_peak": round(gbs / (peak * ctx.world), 4),
                     "us_per_step": round(t_max / steps * 1e6, 3),
                     "gflops": round(w.flops() * steps / t_max / 1e9, 2),
                     "alg_bytes": alg, "launches_per_step": lps, "l2": mode,
                     "scaling": "strong" if ctx.world > 1 else None}
            if mode == "rotate":
                entry["rotating_copies"] = R
            if mode in ("stream", "rotate"):  # also the conservative flushed number
                tf, _ = time_steps(fn, steps, args.warmup, ctx, flush, mode="flush",
                                   charge_writeback=w.op == "ger")
                tfm = ctx.max(sum(tf) / 1000.0)
                entry["flushed_us_per_step"] = round(tfm / steps * 1e6, 3)
                entry["flushed_gbs"] = round(alg * steps / tfm / 1e9, 2)
            # the drop-in call on pinned host buffers for every config that fits
            # a few GiB of host memory (G4 16 GiB and D2 32 GiB per step would
            # add seconds of PCIe per step to the run)
            if (ctx.world == 1 and not fused and not args.no_e2e
                    and w.alg_bytes(1) <= E2E_SUITE_MAX_BYTES):
                a, b = run_e2e(wl, ins, policy, ctx, args, resident=False)
                host = b if b is not None else a  # (resident, host) / (host, None)
                entry["e2e"] = {k: host[k] for k in ("value", "unit", "h2d_bytes_per_step",
                                                     "d2h_bytes_per_step", "ms_per_step")}
                entry["e2e"]["frac_of_link"] = host["link"]["frac_of_link"]
                if "frac_of_duplex_bound" in host["link"]:
                    entry["e2e"]["frac_of_duplex_bound"] = host["link"]["frac_of_duplex_bound"]
                    entry["e2e"]["d2h_gbs_measured"] = host["link"]["d2h_gbs_measured"]
            out[wid] = entry
            del ins
        except torch.cuda.OutOfMemoryError as ex:
            out[wid] = {"error": f"OOM: {ex}"}
        except RuntimeError as ex:  # e.g. no CUDA IPC between the ranks (D2f); agreed on every rank
            if not fused:
                raise
            out[wid] = {"error": f"peer-memory path unavailable: {ex}"}
        torch.cuda.empty_cache()
    return out


# ------------------------------------------------------------ reference arm
def run_reference(args, ctx):
    """The reference's own CPU implementation (compiled oracle/_ref; the
    restated oracle only if the reference build is absent) on all host cores,
    same workload/metric as our arm.  Rank 0 only."""
    if ctx.rank != 0:
        return
    import numpy as np

    from oracle import oracle as O
    from paper_2108_02025_b200 import workloads as WL
    w = WL.WORKLOADS[args.workload]
    cores = os.cpu_count() or 1
    kind = "reference" if O.ref_available() else "port"
    npdt = np.float32 if w.dtype_name == "f32" else np.float64
    gen = lambda n, st: O.gen_uniform(n, npdt, WL.SEED, st)  # noqa: E731
    if w.op == "dot":
        x, y = gen(w.n, WL.STREAM_X), gen(w.n, WL.STREAM_Y)
        sess = O.RefSession("dot", npdt, 0, 0, w.n, None, x, y, 0.0, cores=cores) \
            if kind == "reference" else None
    elif w.op.startswith("gemv"):
        A, x, c = gen(w.m * w.n, WL.STREAM_A), gen(w.n, WL.STREAM_X), gen(w.m, WL.STREAM_C)
        sess = O.RefSession(w.op, npdt, 0 if w.op == "gemv-row" else 1, w.m, w.n, A, x, c,
                            cores=cores) if kind == "reference" else None
    else:
        A, x, c = gen(w.m * w.n, WL.STREAM_CC), gen(w.m, WL.STREAM_X), gen(w.n, WL.STREAM_Y)
        sess = O.RefSession("ger", npdt, 0, w.m, w.n, A, x, c, cores=cores) \
            if kind == "reference" else None

    def one():
        if sess is not None:
            sess.run(False, cores)
        elif w.op == "dot":
            O.dot_ref(x, y, 0.0)
        elif w.op == "ger":
            O.ger_ref(x, c, A, 0)
        else:
            O.gemv_ref(A, 0, x, c)

    # each step is one full pass over the workload; bound the step count so
    # the run stays within a few minutes
    for _ in range(max(1, min(args.warmup, 3))):
        one()
    t_probe = time.perf_counter()
    one()
    per = time.perf_counter() - t_probe
    steps = max(1, min(args.steps, int(120.0 / max(per, 1e-6))))
    t0 = time.perf_counter()
    for _ in range(steps):
        one()
    t = time.perf_counter() - t0
    value = w.alg_bytes(1) * steps / t / 1e9
    used = cores if kind == "reference" else 1
    line = {
        "metric": "DOT/GEMV/GER achieved HBM GB/s & % of B200 roofline at 1/2/4/8 GPUs",
        "impl": "reference",
        "value": round(value, 3), "unit": "GB/s", "n_gpus": ctx.world, "steps": steps,
        "warmup": args.warmup, "ms_per_step": round(t / steps * 1e3, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": w.dtype_name,
        "data": "synthetic: seeded SplitMix64 U[-1,1) (seed 42), generated on the host",
        "config": workload_config(w),
        "run": {"parallelism": f"CPU threads (reference ThreadPool, {used} threads), rank 0 only"},
        "cpu_baseline": {"value": round(value, 3), "unit": "GB/s", "cores": used, "kind": kind,
                         "sample": f"full {w.id} workload per step; "
                                   f"{'cabl::' + w.op.replace('-', '_') if kind == 'reference' else 'restated oracle'}"
                                   f" with ExecPolicy threads={used}"},
        "e2e": {"value": round(value, 3), "unit": "GB/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


def run_cpu_table(args):
    """--cpu-table: the compiled reference on the host cores for every
    BASELINE config at full size: threaded path at
    1 thread and at all cores, and the naive oracle; one JSON line per
    measurement.  Configs whose inputs would not fit 1/3 of free host memory
    are sampled (rows or length cut) and say so."""
    import psutil

    from paper_2108_02025_b200 import workloads as WL
    avail = psutil.virtual_memory().available
    cores = os.cpu_count() or 1
    for wid, w in WL.WORKLOADS.items():
        full = w.alg_bytes(1)
        cap = min(full, avail // 3)
        reps = 5 if full < (1 << 31) else 3
        for label, threads, naive in (("threads=1", 1, False), (f"threads={cores}", cores, False),
                                      ("naive oracle", 1, True)):
            r = cpu_reference_sample(w, max_bytes=cap, reps=reps, threads=threads, naive=naive)
            r.update({"config": wid, "desc": w.desc, "path": label,
                      "full_size": cap >= full})
            print(json.dumps(r), flush=True)


def fail(msg: str, code: int = 3):
    print(f"bench.py: {msg}", file=sys.stderr, flush=True)
    sys.exit(code)


def _free_port() -> int:
    import socket
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def ensure_ranks(args) -> None:
    """One process per GPU.  Under torchrun (WORLD_SIZE set) the world must
    equal --gpus.  Without it, --gpus N > 1 re-executes this command under
    torch.distributed.run with N ranks on this node (127.0.0.1 rendezvous)
    and exits with its status — after checking that N GPUs are visible (our
    arm; the reference arm and --launch-check run on the host)."""
    env_world = os.environ.get("WORLD_SIZE")
    if env_world is not None:
        if int(env_world) != args.gpus:
            fail(f"WORLD_SIZE={env_world} but --gpus {args.gpus}: launch one rank per GPU "
                 f"(torchrun --nproc-per-node {args.gpus}) or drop torchrun and let bench.py "
                 "spawn the ranks")
        return
    if args.gpus == 1:
        return
    if args.impl == "ours" and not args.launch_check and not args.cpu_table:
        import torch
        have = torch.cuda.device_count() if torch.cuda.is_available() else 0
        if have < args.gpus:
            fail(f"--gpus {args.gpus} needs {args.gpus} visible GPUs, found {have}")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={_free_port()}", str(Path(__file__).resolve()), *sys.argv[1:]]
    import subprocess
    sys.exit(subprocess.call(cmd))


def launch_check(world: int, rank: int) -> None:
    """Every rank joins a gloo group and reports itself; rank 0 prints them."""
    ranks = [rank]
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")
        got: list = [None] * world
        dist.all_gather_object(got, {"rank": rank, "pid": os.getpid(),
                                     "local_rank": int(os.environ.get("LOCAL_RANK", "0"))})
        ranks = got
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps({"launch_check": True, "n_gpus": world, "ranks": ranks}), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--cpu-table", action="store_true",
                    help="time the compiled reference on the host for every config and exit")
    ap.add_argument("--workload", default="G1")
    ap.add_argument("--no-suite", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--suite-steps", type=int, default=30)
    ap.add_argument("--suite-timeout", type=float, default=None,
                    help="seconds after which a suite that has not finished is abandoned and "
                         "the headline line printed without it (default: 600 at N > 1, never "
                         "at N = 1; 0 = never)")
    ap.add_argument("--fused-suite", action="store_true",
                    help="at N > 1 also time D2 / G4 with the exchange fused into the kernels "
                         "over peer memory (always on at N = 1)")
    ap.add_argument("--l2", choices=["auto", "flush", "stream"], default="auto",
                    help="headline L2 policy: auto = back to back when a step's inputs "
                         "exceed 2x L2, else flush between steps")
    ap.add_argument("--launch-check", action="store_true",
                    help="spawn the --gpus ranks, rendezvous over gloo, print the rank list and "
                         "exit (CPU; tests the launcher)")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        print("bench.py: --warmup must be >= 3", file=sys.stderr)
        args.warmup = 3
    if args.gpus < 1:
        fail(f"--gpus must be >= 1 (got {args.gpus})")

    ensure_ranks(args)
    world, rank, local = dist_env()
    if args.launch_check:
        launch_check(world, rank)
        return
    if args.cpu_table:
        if rank == 0:
            run_cpu_table(args)
        return
    if args.impl == "reference":
        ctx = Ctx(world, rank, local, None)
        run_reference(args, ctx)
        return

    # a fused peer-memory step whose peer never arrives gives up after 3 s
    # (library default 30 s), so the suite reports it unavailable promptly
    os.environ.setdefault("CABL_PEER_TIMEOUT_MS", "3000")
    import torch
    if not torch.cuda.is_available():
        print(json.dumps({"error": "no CUDA device; libcabl_cuda has no CPU path"}))
        sys.exit(2)
    if local >= torch.cuda.device_count():
        fail(f"rank {rank}: LOCAL_RANK {local} but only {torch.cuda.device_count()} GPU(s) visible")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    ctx = Ctx(world, rank, local, dev)
    try:
        run_ours(args, ctx)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
