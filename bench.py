"""Benchmark of the B200 EBC Greedy hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl ours|reference]

One *step* = one full Greedy(k) run of the configured workload (default C2:
k=50, N=100,000, d=100, fp32, Gaussian seed 1; --config C4 is
the north star's scaling configuration) with V already resident in HBM.
value = point-candidate distance evaluations per second, E = N * sum_{s<k}
(N - s) per run, over all ranks.

Multi-GPU: one rank per GPU.  Under torchrun (WORLD_SIZE set) every rank
builds its own context and the candidates are sharded across ranks (strong
scaling: the same total work), with the per-step exchange on the devices (NCCL
all-gather of 128-B tie-set frontiers) and an end-of-run cross-rank check of
the selection.  ``--gpus N`` without torchrun re-launches itself as N ranks
(torch.distributed.run on 127.0.0.1) and fails if fewer than N GPUs are
visible.

Timing: W untimed warm-up runs; then K runs, each bracketed by a barrier and
device syncs, timed with CUDA events recorded on the library's own stream;
max over ranks.  The timed runs are CUDA-graph replays with the per-step
kernel-family events captured inside the graph (the roofline's screen time).
L2 (126 MB) is flushed before every timed run.  SM clocks are sampled with
nvidia-smi during the timed region.

`e2e` runs the same workload through the public API from host data every
step: EbcFunction(GroundMatrix) (host->device copy of V + baseline) then
greedy_maximize (results device->host), wall-clock.

`--impl reference` times the reference path's CPU implementation -- the fp64
restatement in oracle/ (the reference is pure Python) -- on
the host cores of this box, bounded samples, rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))

import datasets  # noqa: E402

PEAK_FP32_OPS = 148 * 128 * 1.965e9  # FMA-pipe ops/s, SURVEY.md §8(d)
CONFIG_DESC = {
    "C1": "Greedy k=10 EBC, synthetic Gaussian N=2,000 d=16 fp32",
    "C2": "Greedy k=50 EBC, synthetic Gaussian N=100,000 d=100 fp32",
    "C3": "Greedy k=50 EBC, synthetic Gaussian N=100,000 d=100 fp16 storage",
    "C4": "Greedy k=20 EBC, injection-molding surrogate N=500,000 d=32 fp32",
    "C5": "work-matrix evaluation, 4,096 sets x 10 members, synthetic Gaussian N=200,000 d=64 fp32",
    "C4S50": "Greedy k=20 EBC, 50-regime surrogate N=500,000 d=32 fp32 (SURVEY 8(d) near-tie stress case)",
}
METRIC = "Greedy EBC point-candidate distance evals/s (wall time & FMA roofline)"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def evals_per_run(n: int, k: int) -> int:
    return int(n * sum(n - s for s in range(k)))


# ------------------------------------------------------------------ clocks

class ClockSampler:
    """SM clocks and throttle reasons DURING the timed region.  NVML polled from
    a thread every ~1 ms (the timed region of a lazy C2 run is ~15 ms; the
    nvidia-smi loop's 200 ms period never lands inside it), plus one sample at
    start and one at stop; nvidia-smi -lms 200 when NVML is unavailable."""

    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown"}

    def __init__(self, device: int):
        self.device = device
        self.samples = []  # (sm_mhz, sm_max_mhz, reasons bitmask)
        self.stop_evt = threading.Event()
        self.thread = None
        self.nvml = None
        self.proc = None
        self.lines = []

    def _sample(self):
        nv, h = self.nvml
        self.samples.append((nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM),
                             nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM),
                             nv.nvmlDeviceGetCurrentClocksEventReasons(h)))

    def _poll(self):
        while not self.stop_evt.is_set():
            self._sample()
            time.sleep(0.001)

    def start(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            idx = self.device
            vis = os.environ.get("CUDA_VISIBLE_DEVICES", "")
            if vis and vis.replace(",", "").isdigit():
                idx = int(vis.split(",")[self.device])
            self.nvml = (nv, nv.nvmlDeviceGetHandleByIndex(idx))
            self._sample()
            self.thread = threading.Thread(target=self._poll, daemon=True)
            self.thread.start()
            return
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
                 "--format=csv,noheader,nounits", "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                text=True)
            self.thread = threading.Thread(target=lambda: self.lines.extend(ln.strip() for ln in self.proc.stdout),
                                           daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None

    def stop(self):
        if self.nvml is not None:
            self._sample()
            self.stop_evt.set()
            self.thread.join(timeout=2)
            rows = self.samples
        elif self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            rows = []
            for ln in self.lines:
                parts = [p.strip() for p in ln.split(",")]
                try:
                    rows.append((float(parts[0]), float(parts[1]), int(parts[2], 16)))
                except (ValueError, IndexError):
                    pass
        else:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no clock source"], "samples": 0}
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        sm = [r[0] for r in rows]
        reasons = sorted({name for r in rows for bit, name in self.REASONS.items() if r[2] & bit})
        loaded = [x for x in sm if x > 0.5 * max(sm)]
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": max(r[1] for r in rows), "reasons": reasons,
                "samples": len(rows), "source": "nvml" if self.nvml is not None else "nvidia-smi"}


# ------------------------------------------------------------------ helpers

def flush_l2(torch, dev):
    buf = getattr(flush_l2, "_buf", None)
    if buf is None or buf.device != dev:
        buf = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
        flush_l2._buf = buf
    buf.fill_(1.0)


# tcgen05.ld bytes per clock per SM with 8 loading warps, measured on B200
# (tools/microbench/tmem_ld.cu -> profiles/r01_microbench_tmem_ld.txt)
TMEM_LD_BPC = 335.0


def load_measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            return json.load(fh)
    except (OSError, ValueError):
        return None


def load_profile_traffic(config: str):
    """dram bytes per launch of k_screen from the committed ncu --set full summary."""
    path = os.path.join(ROOT, "profiles", "screen_ncu_summary.json")
    if not os.path.exists(path):
        return None, None
    with open(path) as fh:
        p = json.load(fh)
    c = p.get("configs", {}).get(config)
    if not c:
        return None, None
    return c.get("dram_bytes_per_launch"), c


def cpu_sample(V: np.ndarray, threads: int, target_s: float):
    """Reference CPU path (oracle port) on a bounded candidate prefix of one
    Greedy step: returns (evals/s, description)."""
    import oracle
    oracle.set_threads(threads)
    n = V.shape[0]
    m = 64
    while True:
        t0 = time.perf_counter()
        oracle.step_values(V, [], range(m))
        dt = time.perf_counter() - t0
        if dt >= target_s or m >= n:
            break
        m = min(n, max(m * 2, int(m * target_s / max(dt, 1e-3) * 1.1)))
    return n * m / dt, f"first Greedy step, candidates [0,{m}) x all {n} points, {dt:.1f}s"


def workload(config: str):
    X = datasets.config_data(config)
    k = datasets.CONFIG_K[config]
    return X, k


# ------------------------------------------------------------------ reference arm

def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    if args.config == "C5":
        import oracle
        X, sets = datasets.c5_problem()
        threads = len(os.sched_getaffinity(0))
        oracle.set_threads(threads)
        V = X.astype(np.float64)
        rates = []
        for i in range(args.warmup + args.steps):
            m = 64 if i < args.warmup else 512
            t0 = time.perf_counter()
            oracle.eval_multiset(V, sets[:m])
            dt = time.perf_counter() - t0
            if i >= args.warmup:
                rates.append(X.shape[0] * 10 * m / dt)
        value = float(np.median(rates))
        work = float(X.shape[0]) * sum(len(x) for x in sets)
        print(json.dumps({
            "impl": "reference", "metric": "work-matrix point-member distance evals/s", "value": value,
            "unit": "point-member evals/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * work / value, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (seeded Gaussian, tests/golden/datasets.c5_problem)",
            "config": {"workload": CONFIG_DESC["C5"], "config_id": "C5", "parallelism": "host threads"},
            "cpu_baseline": {"value": value, "unit": "point-member evals/s", "cores": threads, "kind": "port",
                             "sample": "first 512 sets of the 4,096 per step"},
            "e2e": {"value": value, "unit": "point-member evals/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}), flush=True)
        return 0
    X, k = workload(args.config)
    V = X.astype(np.float64)
    n = V.shape[0]
    threads = len(os.sched_getaffinity(0))
    import oracle
    oracle.build()
    per_step_target = float(os.environ.get("EBC_REF_STEP_SECONDS", "8"))
    rates = []
    desc = ""
    for i in range(args.warmup + args.steps):
        r, desc = cpu_sample(V, threads, per_step_target if i >= args.warmup else 1.0)
        if i >= args.warmup:
            rates.append(r)
    value = float(np.median(rates))
    E = evals_per_run(n, k)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "point-candidate evals/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * E / value, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, tests/golden/datasets.py)",
        "config": {"workload": CONFIG_DESC.get(args.config, args.config), "config_id": args.config,
                   "N": n, "d": V.shape[1], "k": k, "parallelism": "host threads",
                   "extrapolation": "ms_per_step = full-run evaluations / sampled rate (cached-min step cost is "
                                    "independent of s)"},
        "cpu_baseline": {"value": value, "unit": "point-candidate evals/s", "cores": threads, "kind": "port",
                         "sample": desc},
        "e2e": {"value": value, "unit": "point-candidate evals/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ our arm

def tensor_roofline(info, rung, d, work_pairs, screen_ms, E):
    """Roofline object of the tensor screen: 2 P d flops per evaluated pair (P
    products) over the screen's own time, against the measured BF16 peak."""
    kind = 3 if rung == 0 else int(info[2])
    kname = {0: "3xTF32 kind::tf32", 1: "BF16x3 kind::f16", 2: "FP16x1 kind::f16",
             3: "FP16x1-rounded kind::f16"}[kind]
    nprod = 1 if kind in (2, 3) else 3
    peaks = load_measured_peaks()
    # the screen runs inside a long step (a whole Greedy run, >= 100 ms of
    # back-to-back launches): the SUSTAINED measured BF16 figure is its peak
    # (B200_PROFILING / task contract); the burst figure is reported beside it
    burst = peaks.get("bf16_tflops") if peaks else None
    sust = peaks.get("bf16_tflops_sustained") if peaks else None
    bf16 = sust or burst
    base = bf16 if bf16 else 1590.0
    tpeak = base / 2.0 if kind == 0 else base
    wexec = float(work_pairs) if work_pairs and work_pairs > 0 else float(E)
    tach = 2.0 * nprod * d * wexec / (screen_ms * 1e-3) / 1e12
    return {
        "bound": "tensor",
        "kernel": "k_screen_tc (tcgen05 %s anchored Gram screen, TMEM operands and accumulators)" % kname,
        "achieved": tach, "peak": tpeak, "unit": "TFLOP/s", "frac": tach / tpeak,
        "peak_burst": (burst / 2.0 if kind == 0 else burst) if burst else None,
        "frac_vs_burst": (tach / (burst / 2.0 if kind == 0 else burst)) if burst else None,
        "peak_source": (("MEASURED_PEAKS.json bf16_tflops_sustained" if sust else
                         "MEASURED_PEAKS.json bf16_tflops") if bf16 else "fallback 1.59 PF bf16")
                       + (" / 2 (TF32)" if kind == 0 else "") + "; nominal dense BF16 = 2250 TFLOP/s",
        "work": "%dd tensor flops per evaluated point-candidate pair (%d product%s, d not padded)"
                % (2 * nprod, nprod, "s of the split" if nprod > 1 else " of the fp16 values"),
        "pairs_evaluated": wexec, "pairs_evaluated_frac_of_E": wexec / E,
        "tmem_read": {"achieved": 4.0 * wexec / (screen_ms * 1e-3) / 1e9,
                      "peak": TMEM_LD_BPC * 148 * 1.965e9 / 1e9, "unit": "GB/s",
                      "frac": (4.0 * wexec / (screen_ms * 1e-3)) / (TMEM_LD_BPC * 148 * 1.965e9),
                      "work": "4 B fp32 accumulator per point-candidate pair; peak = tcgen05.ld throughput "
                              "measured with 8 loading warps per SM (the screen's epilogue), "
                              "335 B/clk/SM x 148 SM x 1.965 GHz (profiles/r01_microbench_tmem_ld.txt)"},
        "screen_rung": rung,
        "screen_info": {"mode": info[0], "tile_points": info[1],
                        "operands": {0: "tf32 split", 1: "bf16 split", 2: "fp16",
                                     3: "fp32 rounded to fp16 (scaled)"}[kind], "kpad": info[3]},
    }


def screen_roofline(info, rung, d, work_pairs, screen_ms, step_ms, E, config):
    """Roofline of the dominant kernel (the candidate screen) for one GPU's share
    of the run: its evaluated pairs over its own time (CUDA events on the
    library stream inside the timed region)."""
    achieved = 2.0 * d * E / (screen_ms * 1e-3)
    fma_equiv = {"achieved": achieved / 1e12, "peak": PEAK_FP32_OPS / 1e12, "unit": "TFLOP/s",
                 "frac": achieved / PEAK_FP32_OPS,
                 "work": "W = 2d FP32 FMA-pipe ops per point-candidate pair (SURVEY.md §8(d)), not redefined; "
                         "peak = 148 SM x 128 lanes x 1.965 GHz (nominal)"}
    traffic, _prof = load_profile_traffic(config)
    if rung in (0, 1):
        line = tensor_roofline(info, rung, d, work_pairs, screen_ms, E)
        line["traffic"] = traffic
        line["fma_equiv"] = dict(fma_equiv, flag="frac > 1.0 expected: tensor cores vs the FP32 FMA roofline")
    else:
        line = {"bound": "fma", "kernel": "k_screen (fused distance->min->sum on the FP32 FMA pipe)",
                "achieved": fma_equiv["achieved"], "peak": fma_equiv["peak"], "unit": "TFLOP/s",
                "frac": fma_equiv["frac"], "traffic": traffic, "work": fma_equiv["work"],
                "flag": ("frac > 1.0: the Gram rung issues d FFMA per pair against the direct-form W = 2d"
                         if achieved > PEAK_FP32_OPS else None), "screen_rung": rung}
    line["screen_ms_per_step"] = screen_ms
    line["screen_share_of_step"] = screen_ms / step_ms
    return line


def update_roofline(n_pts, d, k, update_ms):
    """Second ceiling named by the north star: the cached-min update (K4) is
    HBM-bound; algorithmic bytes per step = N (4 pitch + 8 cm + 8 e0d + 8 term)
    (the seed refresh of changed points and the fused batch's term traffic not
    counted), against the measured HBM copy bandwidth; its time is the update
    family per step (CUDA events): on lazy runs k_update_batch alone (the
    cached-min update fused with the next step's first batch refine; the
    batch's top-k is timed with the selection)."""
    peaks = load_measured_peaks()
    hbm = (peaks or {}).get("hbm_gbs")
    per_step_ms = update_ms / k
    pitch = (d + 3) // 4 * 4
    if (pitch // 4) % 2 == 0:
        pitch += 4
    ubytes = n_pts * (4.0 * pitch + 24.0)
    ach = ubytes / (per_step_ms * 1e-3) / 1e9
    return {"bound": "hbm", "kernel": "k_update_batch (cached-min update + fixed-order f(S) + the next step's first "
                                      "batch refine, one launch; k_update_fused on non-lazy steps)",
            "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": (ach / hbm) if hbm else None,
            "bytes_per_step": ubytes, "us_per_step": per_step_ms * 1e3,
            "peak_source": "MEASURED_PEAKS.json hbm_gbs" if hbm else None,
            "note": "V may be partly L2-resident between steps (40-64 MB vs 126 MB L2); algorithmic bytes, "
                    "not DRAM bytes"}


def run_ours(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    ndev = torch.cuda.device_count()
    if ndev < 1:
        raise RuntimeError("bench.py needs a CUDA device (the b200 path has no CPU fallback)")
    if world != args.gpus:
        raise RuntimeError(f"--gpus {args.gpus} but WORLD_SIZE={world}: launch one rank per GPU")
    shared_gpu = os.environ.get("EBC_BENCH_SHARE_GPU") == "1"
    if world > ndev and not shared_gpu:
        raise RuntimeError(f"{world} ranks but only {ndev} visible GPU(s): one rank per GPU "
                           f"(EBC_BENCH_SHARE_GPU=1 runs the gloo test mode)")
    dev_index = local_rank % ndev
    torch.cuda.set_device(dev_index)
    dev = torch.device("cuda", dev_index)
    distributed = world > 1
    if distributed:
        backend = "nccl" if world <= ndev else "gloo"  # gloo only in the shared-GPU test mode
        dist.init_process_group(backend, device_id=dev if backend == "nccl" else None)
    os.environ["EBC200_DEVICE"] = str(dev_index)
    nccl = distributed and dist.get_backend() == "nccl"

    import paper_2105_12026_b200 as eb
    from paper_2105_12026_b200 import optimize
    from paper_2105_12026_b200.sharded import greedy_maximize_sharded

    X, k = workload(args.config)
    n, d = X.shape
    prec = eb.Precision.FP16_STORAGE if X.dtype == np.float16 else eb.Precision.FP32
    g = eb.GroundMatrix(X, prec)
    f = eb.EbcFunction(g, device=dev_index)
    lib_stream = torch.cuda.ExternalStream(f._lib.ebc_stream(f.native_context), device=dev)
    budget = eb.OptimizerBudget(k=k)

    def one_run(fx=f):
        if distributed:
            return greedy_maximize_sharded(fx, budget)
        return eb.greedy_maximize(fx, budget)

    def barrier():
        if distributed:
            dist.barrier()

    def timed(fx, runs, families):
        """`runs` graph replays of fx, each after an L2 flush, bracketed by
        barriers + syncs, CUDA events on the library stream."""
        ms, scr, upd, wk, st, launches, last = [], [], [], [], None, 0, None
        for _ in range(runs):
            flush_l2(torch, dev)
            torch.cuda.synchronize(dev)
            barrier()
            ev0 = torch.cuda.Event(enable_timing=True)
            ev1 = torch.cuda.Event(enable_timing=True)
            ev0.record(lib_stream)
            last = one_run(fx)
            ev1.record(lib_stream)
            torch.cuda.synchronize(dev)
            barrier()
            ms.append(ev0.elapsed_time(ev1))
            # NCCL path: the whole run is one native call (graph); host-driven
            # (gloo) path: the count of the last per-step native call
            launches += optimize.last_launches(fx)
            if families:
                t = optimize.last_timings(fx)
                scr.append(t[0])
                upd.append(t[2])
                st = optimize.last_stats(fx)
                wk.append(optimize.last_screen_work(fx))
            if ref_sel is not None and last.selected != ref_sel:
                raise RuntimeError("selection changed between runs")
        return ms, scr, upd, wk, st, launches, last

    # (a) the product path as a user runs it (lazy steps, no timing events in
    # the graph): ms_per_step / value
    ref_sel = None
    for _ in range(args.warmup):
        ref_sel = one_run().selected
    clocks = ClockSampler(dev_index)
    clocks.start()
    times_ms, _, _, _, _, launches, s = timed(f, args.steps, False)
    clk = clocks.stop()
    timed_families = (not distributed) or nccl
    lazy = optimize.last_lazy_stats(f)
    # (b) the same runs with per-step family events captured in the graph:
    # selection vs cached-min update time (update_roofline)
    optimize.set_timing(f, True)
    for _ in range(3):
        one_run()
    _, sel_ms, update_ms, _, stats, _, _ = timed(f, 2, timed_families)
    optimize.set_timing(f, False)
    # (c) the dominant kernel's roofline: the tensor screen measured on a
    # context whose every step screens every candidate (EBC200_LAZY=0; the lazy
    # run screens fully only at step 0 and in re-screened steps), and that
    # run's time for reference
    os.environ["EBC200_LAZY"] = "0"
    try:
        fk = eb.EbcFunction(g, device=dev_index)
    finally:
        del os.environ["EBC200_LAZY"]
    optimize.set_timing(fk, True)
    for _ in range(3):
        one_run(fk)
    full_ms, screen_ms, _, work, full_stats, _, sk = timed(fk, 2, timed_families)
    if sk.selected != s.selected or sk.value != s.value:
        raise RuntimeError("lazy and full-screen runs disagree")
    fk.close()

    E = evals_per_run(n, k)
    mine = {"step_ms": float(np.mean(times_ms)), "launches": int(launches),
            "screen_ms": float(np.mean(screen_ms)) if screen_ms else None,
            "update_ms": float(np.mean(update_ms)) if update_ms else None,
            "sel_ms": float(np.mean(sel_ms)) if sel_ms else None,
            "full_ms": float(np.mean(full_ms)), "full_stats": full_stats,
            "work": float(np.mean(work)) if work else None, "stats": stats, "lazy": lazy,
            "selected": s.selected, "value": s.value}

    # e2e through the public API from host data: EbcFunction(GroundMatrix) (V
    # host->device) + greedy_maximize(_sharded) (results device->host), wall clock
    e2e_ms = []
    h2d = X.nbytes + d * 8
    d2h = k * 3 * 8 + 8
    for i in range(max(1, min(args.steps, 3))):
        barrier()
        t0 = time.perf_counter()
        f2 = eb.EbcFunction(g, device=dev_index)
        one_run(f2)
        t1 = time.perf_counter()
        barrier()
        e2e_ms.append((t1 - t0) * 1e3)
        f2.close()
    mine["e2e_ms"] = float(np.median(e2e_ms))

    ranks = [mine]
    if distributed:
        ranks = [None] * world
        dist.all_gather_object(ranks, mine)
    if any(r["selected"] != mine["selected"] or r["value"] != mine["value"] for r in ranks):
        raise RuntimeError("ranks disagree on the selection")

    if rank != 0:
        if distributed:
            dist.destroy_process_group()
        return 0

    step_ms = max(r["step_ms"] for r in ranks)  # device time, max over ranks
    e2e_step = max(r["e2e_ms"] for r in ranks)
    value = E / (step_ms * 1e-3)
    line = {
        "metric": METRIC, "value": value, "unit": "point-candidate evals/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32" if prec is eb.Precision.FP32 else "f16-storage/f32",
        "data": "synthetic (seeded Gaussian / surrogate, tests/golden/datasets.py)",
        "config": {"workload": CONFIG_DESC[args.config], "config_id": args.config, "N": n, "d": d, "k": k,
                   "evals_per_step": E,
                   "parallelism": (f"candidate-sharded x{world} ({'NCCL device exchange' if nccl else 'gloo host exchange'})"
                                   if distributed else "1 GPU"),
                   "l2": "flushed (256 MB write) before every timed run; V is 40-64 MB",
                   "timed_runs": "CUDA-graph replays of the product path (no timing events in the graph); "
                                 "kernel-family times and the screen roofline from separate event-instrumented "
                                 "replays"},
        "selected_head": s.selected[:5], "summary_value": s.value,
        "clocks": clk,
        "e2e": {"value": E / (e2e_step * 1e-3), "unit": "point-candidate evals/s", "ms_per_step": e2e_step,
                "h2d_bytes_per_step": int(h2d) * world, "d2h_bytes_per_step": int(d2h) * world,
                "path": "EbcFunction(GroundMatrix) + greedy_maximize%s via libebc200.so C-ABI; host rows page-locked (the GroundMatrix's buffer, registered at its first context), results to pageable host memory"
                        % ("_sharded (every rank uploads V)" if distributed else "")},
        "gpu_launches": int(sum(r["launches"] for r in ranks)),
    }
    if distributed:
        line["per_rank_ms_per_step"] = [r["step_ms"] for r in ranks]
    if timed_families and all(r["screen_ms"] for r in ranks):
        info = optimize.screen_info(f)
        # one GPU's share: the slowest rank's screen over that rank's own pairs,
        # measured on the full-screen (EBC200_LAZY=0) run of the same workload
        slow = max(range(world), key=lambda r: ranks[r]["screen_ms"])
        rr = ranks[slow]
        fst = rr["full_stats"]
        rung = fst[2] if fst else -1
        e_rank = E / world
        line["roofline"] = screen_roofline(info, rung, d, rr["work"], rr["screen_ms"], rr["full_ms"], e_rank,
                                           args.config)
        line["roofline"]["measured_on"] = ("full-screen run of the same workload (EBC200_LAZY=0: every step screens "
                                           "every candidate); the product run screens fully at step 0 and in "
                                           "re-screened lazy steps only")
        if distributed:
            line["roofline"]["rank"] = slow
            line["roofline"]["per_rank_frac"] = [
                screen_roofline(info, (q["full_stats"] or [0, 0, -1])[2], d, q["work"], q["screen_ms"], q["full_ms"],
                                e_rank, args.config)["frac"] for q in ranks]
        line["window"] = {"sum": rr["stats"][0], "max": rr["stats"][1], "steps": rr["stats"][3]} if rr["stats"] else None
        if rr["update_ms"]:
            line["update_roofline"] = update_roofline(n, d, k, rr["update_ms"])
    lz = mine["lazy"]
    line["lazy"] = {
        "enabled": bool(lz[0]), "lazy_steps": lz[1], "decided_without_screen": lz[2],
        "candidates_reexamined": lz[3],
        "full_screen_ms_per_step": max(r["full_ms"] for r in ranks),
        "speedup_vs_full_screen": max(r["full_ms"] for r in ranks) / step_ms,
        "rule": "a step re-examines only candidates whose last certified bound (screen upper bound or exact gain) "
                "can still reach the reference tie window (gains only shrink: f is submodular); selections, values "
                "and gains are bit-identical to the full-screen run (checked here and in tests)",
    }
    if not args.no_cpu_baseline:
        threads = len(os.sched_getaffinity(0))
        rate, desc = cpu_sample(X.astype(np.float64), threads, float(os.environ.get("EBC_CPU_SECONDS", "10")))
        line["cpu_baseline"] = {"value": rate, "unit": "point-candidate evals/s", "cores": threads,
                                "kind": "port", "sample": desc}
    print(json.dumps(line), flush=True)
    if distributed:
        dist.destroy_process_group()
    return 0


def run_multiset(args):
    """C5: one step = one evaluate_with_backend of the 4,096-set work matrix
    (batched.py:180-240); N > 1: the sets split across ranks
    (evaluate_multiset_sharded, fp64 values all-gathered)."""
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    ndev = torch.cuda.device_count()
    if ndev < 1:
        raise RuntimeError("bench.py needs a CUDA device (the b200 path has no CPU fallback)")
    dev_index = local_rank % ndev
    torch.cuda.set_device(dev_index)
    dev = torch.device("cuda", dev_index)
    distributed = world > 1
    if distributed:
        backend = "nccl" if world <= ndev else "gloo"
        dist.init_process_group(backend, device_id=dev if backend == "nccl" else None)
    os.environ["EBC200_DEVICE"] = str(dev_index)
    import paper_2105_12026_b200 as eb
    from paper_2105_12026_b200 import optimize
    from paper_2105_12026_b200.sharded import evaluate_multiset_sharded

    X, sets = datasets.c5_problem()
    n, d = X.shape
    g = eb.GroundMatrix(X, eb.Precision.FP32)
    f = eb.EbcFunction(g, device=dev_index)
    ms = eb.EvalMultiset(sets)
    lib_stream = torch.cuda.ExternalStream(f._lib.ebc_stream(f.native_context), device=dev)

    def one(fx=f):
        return evaluate_multiset_sharded(fx, ms) if distributed else eb.evaluate_with_backend(fx, ms)

    def barrier():
        if distributed:
            dist.barrier()

    ref = None
    for _ in range(args.warmup):
        ref = one()
    clocks = ClockSampler(dev_index)
    clocks.start()
    times, launches = [], 0
    for _ in range(args.steps):
        flush_l2(torch, dev)
        torch.cuda.synchronize(dev)
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(lib_stream)
        vals = one()
        e1.record(lib_stream)
        torch.cuda.synchronize(dev)
        barrier()
        times.append(e0.elapsed_time(e1))
        launches += optimize.last_launches(f)
        if not np.array_equal(vals, ref):
            raise RuntimeError("values changed between runs")
    clk = clocks.stop()
    e2e = []
    for _ in range(max(1, min(args.steps, 3))):
        barrier()
        t0 = time.perf_counter()
        f2 = eb.EbcFunction(g, device=dev_index)
        one(f2)
        e2e.append((time.perf_counter() - t0) * 1e3)
        barrier()
        f2.close()
    mine = {"ms": float(np.mean(times)), "e2e": float(np.median(e2e)), "launches": launches}
    ranks = [mine]
    if distributed:
        ranks = [None] * world
        dist.all_gather_object(ranks, mine)
    if rank != 0:
        if distributed:
            dist.destroy_process_group()
        return 0
    ms_step = max(r["ms"] for r in ranks)
    e2e_step = max(r["e2e"] for r in ranks)
    work = float(n) * sum(len(x) for x in sets)  # point-member distance evaluations per step
    line = {
        "metric": "work-matrix point-member distance evals/s", "value": work / (ms_step * 1e-3),
        "unit": "point-member evals/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic (seeded Gaussian, tests/golden/datasets.c5_problem)",
        "config": {"workload": CONFIG_DESC["C5"], "config_id": "C5", "N": n, "d": d, "sets": len(sets),
                   "members": 10, "parallelism": f"set-sharded x{world}" if distributed else "1 GPU",
                   "l2": "flushed (256 MB write) before every timed call",
                   "timed_runs": "whole evaluate_with_backend calls (CSR upload, device work, values back)"},
        "clocks": clk,
        "e2e": {"value": work / (e2e_step * 1e-3), "unit": "point-member evals/s", "ms_per_step": e2e_step,
                "h2d_bytes_per_step": int(X.nbytes + 8 * (len(sets) + 1 + sum(len(x) for x in sets))),
                "d2h_bytes_per_step": 8 * len(sets)},
        "gpu_launches": int(sum(r["launches"] for r in ranks)),
        "roofline": None,
        "roofline_note": "dominant kernel: the tensor flag screen (profiles/r01_screen_tc_flag_c5_ncu_summary.txt)",
    }
    if not args.no_cpu_baseline:
        import oracle
        threads = len(os.sched_getaffinity(0))
        oracle.set_threads(threads)
        m = 256
        t0 = time.perf_counter()
        oracle.eval_multiset(X.astype(np.float64), sets[:m])
        dt = time.perf_counter() - t0
        line["cpu_baseline"] = {"value": n * 10 * m / dt, "unit": "point-member evals/s", "cores": threads,
                                "kind": "port", "sample": f"first {m} sets, {dt:.1f}s"}
    print(json.dumps(line), flush=True)
    if distributed:
        dist.destroy_process_group()
    return 0


def spawn_ranks(args, argv):
    """--gpus N > 1 outside torchrun: re-launch this script as N ranks, one per
    GPU (torch.distributed.run on 127.0.0.1); refuses to oversubscribe GPUs."""
    import socket

    import torch
    ndev = torch.cuda.device_count()
    if args.gpus > ndev and os.environ.get("EBC_BENCH_SHARE_GPU") != "1":
        log(f"error: --gpus {args.gpus} needs {args.gpus} GPUs, {ndev} visible")
        return 2
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *argv]
    return subprocess.call(cmd)


def main(argv=None):
    ap = argparse.ArgumentParser(description=__doc__.splitlines()[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default=os.environ.get("EBC_BENCH_CONFIG", "C2"), choices=sorted(CONFIG_DESC))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    raw = list(sys.argv[1:] if argv is None else argv)
    args = ap.parse_args(raw)
    if args.gpus < 1:
        ap.error("--gpus must be >= 1")
    if args.warmup < 3:
        log("note: warm-up raised to the contract minimum of 3")
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args, raw)
    if args.config == "C5":
        return run_multiset(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
