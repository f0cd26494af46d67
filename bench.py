"""Benchmark of the B200 IMM hot path (one JSON line on rank 0).

Workload (default): BASELINE.json configs[4] (c5), the largest single-GPU config -- BASELINE's
metric names no config, so the N=1 line is quoted on the largest one: directed R-MAT scale 25
(33.5 M vertices), edge factor 42 (1.37 B edges after dedup), (a,b,c,d)=(0.57,0.19,0.19,0.05),
generator seed 4, weighted-cascade IC fl32(1/indeg(v)), IMM k=50, epsilon=0.5, 8 blocks,
per-set hybrid store (Huffman; bitmap for sets above n/32), sampling seed 42.  `--config
c1..c4` runs the others.  Synthetic data: the paper's SNAP/LAW graphs are not available.

A step = one full IMM run (theta estimation -> sampling + learn-then-compress encoding ->
greedy selection on the compressed store).  `value` = RRR samples materialised per second
of the step, graph resident in HBM; `e2e` = the same through the C-ABI from pinned host
buffers (forward graph H2D + device transpose + run + results D2H inside the timed region).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5] [--impl ours|reference]

N > 1: one process per GPU under torchrun; replicas only (the path has no data exchange at
this tier), value = samples of all ranks / max-over-ranks time.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (generator, weights, k, eps, blocks, mode, description)
    "c1": dict(gen=("er", 10000, 100000, 0), weights=("wc", 0.0), k=10, eps=0.5, blocks=10, mode="huffman", ref_samples=20000,
               desc="ER n=10k m=100k seed 0, WC fl32, k=10 eps=0.5 b=10 huffman"),
    "c2": dict(gen=("rmat", 18, 16, 1), weights=("uniform", 0.01), k=50, eps=0.5, blocks=8, mode="huffman", ref_samples=20000,
               desc="R-MAT scale 18 EF16 (.57,.19,.19) seed 1, IC p=fl32(0.01), k=50 eps=0.5 b=8 huffman"),
    "c3": dict(gen=("rmat", 20, 16, 2), weights=("wc", 0.0), k=100, eps=0.5, blocks=8, mode="hybrid",
               desc="R-MAT scale 20 EF16 seed 2, LT (in-weights U(0,1) normalised, f32, seed 3), k=100 eps=0.5 b=8 "
                    "per-set hybrid (bitmap above n/32, Huffman otherwise)", device_gen=True, lt_seed=3,
               ref_samples=20000),
    "c4": dict(gen=("rmat", 22, 24, 3), weights=("wc", 0.0), k=100, eps=0.13, blocks=8, mode="huffman",
               desc="R-MAT scale 22 EF24 seed 3, WC fl32, k=100 eps=0.13 b=8 huffman", device_gen=True,
               ref_samples=20000),
    "c5": dict(gen=("rmat", 25, 42, 4), weights=("wc", 0.0), k=50, eps=0.5, blocks=8, mode="hybrid",
               desc="R-MAT scale 25 EF42 seed 4, WC fl32, k=50 eps=0.5 b=8 per-set hybrid (bitmap above n/32, "
                    "Huffman otherwise)", device_gen=True, ref_samples=4000),
}
DTYPE = "u32/u64 integer (RNG u64, ids u32)"
METRIC = "RRR samples/s & achieved HBM GB/s at 1 B200; IMM end-to-end s; compress ratio"
SEED = 42


def make_graph(im, cfg):
    gen = cfg["gen"]
    if gen[0] == "er":
        g = im.generate_er(gen[1], gen[2], gen[3])
    else:
        g = im.generate_rmat(gen[1], gen[2], 0.57, 0.19, 0.19, gen[3])
    model, p = cfg["weights"]
    im.assign_weights_f32(g, model, p)
    return g


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class NvmlClockSampler:
    """SM clock + clock-event (throttle) reasons polled through NVML in a thread of this
    process during the timed region.  (An `nvidia-smi -lms` child stalled the driver for tens
    of ms per query -- c2 +60..140 ms a step; NVML's two queries do not.)"""

    REASONS = [("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap")]

    def __init__(self, gpu: int, period_ms: int = 200):
        import pynvml as N

        self.N, self.rows, self.period_ms, self.late = N, [], period_ms, False
        N.nvmlInit()
        self.h = None
        try:  # the CUDA device's NVML handle (indices differ under CUDA_VISIBLE_DEVICES)
            import torch

            uuid = str(torch.cuda.get_device_properties(gpu).uuid)
            self.h = N.nvmlDeviceGetHandleByUUID(uuid if uuid.startswith("GPU-") else "GPU-" + uuid)
        except Exception:
            self.h = N.nvmlDeviceGetHandleByIndex(gpu)
        self.max_mhz = float(N.nvmlDeviceGetMaxClockInfo(self.h, N.NVML_CLOCK_SM))
        self.stop = threading.Event()

    def _poll(self):
        N = self.N
        while not self.stop.is_set():
            try:
                mhz = float(N.nvmlDeviceGetClockInfo(self.h, N.NVML_CLOCK_SM))
                rs = N.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.rows.append((mhz, rs))
            except Exception:
                pass
            self.stop.wait(self.period_ms / 1000.0)

    def __enter__(self):
        self.t = threading.Thread(target=self._poll, daemon=True)
        self.t.start()
        return self

    def wait_first(self, timeout: float = 10.0):
        t0 = time.time()
        while not self.rows and time.time() - t0 < timeout:
            time.sleep(0.01)
        self.rows.clear()

    def ensure_one(self):
        self.late = not self.rows
        t0 = time.time()
        while not self.rows and time.time() - t0 < self.period_ms / 1000.0 + 1.0:
            time.sleep(0.01)

    def __exit__(self, *a):
        self.stop.set()
        self.t.join(timeout=2)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"], "samples": 0}
        N = self.N
        reasons = sorted({name for _, rs in self.rows for name, attr in self.REASONS
                          if hasattr(N, attr) and rs & getattr(N, attr)})
        out = {"sm_mhz": float(np.median([m for m, _ in self.rows])), "sm_max_mhz": self.max_mhz,
               "reasons": reasons, "samples": len(self.rows), "period_ms": self.period_ms, "source": "nvml"}
        if self.late:
            out["sampled"] = "right after the timed region (shorter than the sampling period)"
        return out


class NoClockSampler:
    """BENCH_CLOCKS=off: no queries at all (diagnosis of the samplers' own cost only -- a line
    without clocks does not meet the bench contract)."""

    rows, late = [], False

    def __enter__(self):
        return self

    def __exit__(self, *a):
        pass

    def wait_first(self, timeout: float = 10.0):
        pass

    def ensure_one(self):
        pass

    def summary(self):
        return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled (BENCH_CLOCKS=off)"], "samples": 0}


def clock_sampler(gpu: int, period_ms: int):
    """NVML in-process when available (BENCH_CLOCKS=smi forces the nvidia-smi child)."""
    mode = os.environ.get("BENCH_CLOCKS", "nvml")
    if mode == "off":
        return NoClockSampler()
    if mode != "smi":
        try:
            return NvmlClockSampler(gpu, period_ms)
        except Exception:
            pass
    return ClockSampler(gpu, period_ms)


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap"]

    def __init__(self, gpu: int, period_ms: int = 200):
        self.gpu, self.rows, self.proc, self.period_ms = gpu, [], None, period_ms

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), "--query-gpu=" + ",".join(self.FIELDS), "--format=csv,noheader,nounits",
                 "-lms", str(self.period_ms)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def wait_first(self, timeout: float = 10.0):
        # nvidia-smi's start-up (driver/NVML init) is slow and can stall the context: let it
        # finish before the timed region opens, then keep only the samples taken inside it
        t0 = time.time()
        while self.proc and not self.rows and time.time() - t0 < timeout:
            time.sleep(0.02)
        self.rows.clear()

    def ensure_one(self):
        # a timed region shorter than the sampling period takes the next sample
        self.late = not self.rows
        timeout = self.period_ms / 1000.0 + 1.0
        t0 = time.time()
        while self.proc and not self.rows and time.time() - t0 < timeout:
            time.sleep(0.01)

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == len(self.FIELDS):
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i].lower().startswith("active")})
        out = {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
               "reasons": reasons, "samples": len(self.rows), "period_ms": self.period_ms}
        if getattr(self, "late", False):
            out["sampled"] = "right after the timed region (shorter than the sampling period)"
        return out


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def max_over_ranks(x: float, world: int, backend_dev=None) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x: float, world: int, backend_dev=None) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


# ------------------------------------------------------------------ CPU arms
def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


class ReferenceWindow:
    """The reference's CPU sampling path on the workload's graph, loaded from oracle/ only.

    IC configs: the unmodified reference (oracle/_ref/libimmx_ref.so, built from its sources
    with OpenMP) -- G^T is generated inside that library by oracle/gen_graph.c (the same
    definition as the product's device generator, pinned by tests/test_gen_oracle.py and the
    graph SHA-256 goldens), and `sample_block` (sampler.cpp:85-104, the ~99% phase of the
    reference IMM on these configs) samples windows of global indices with all host threads.
    LT (c3): the reference has no LT sampler, so the C restatement's LT walk
    (oracle/liboracle.so oc_sample_block_lt, one thread) is the "port" baseline.
    No product code is loaded on this path."""

    def __init__(self, cfg):
        self.cfg = cfg
        self.lt = "lt_seed" in cfg
        t0 = time.perf_counter()
        if self.lt:
            from oracle.oracle import Oracle

            self.orc = Oracle()
            self.g, self.w = self.orc.generate(cfg["gen"], cfg["weights"], reverse=True, lt_seed=cfg["lt_seed"])
            self.kind, self.threads = "port", 1
        else:
            from oracle.oracle import RefLib

            self.g = RefLib().generate(cfg["gen"], cfg["weights"], reverse=True)
            self.kind, self.threads = "reference", host_cores()
        self.gen_s = time.perf_counter() - t0

    def sample(self, count: int, first: int) -> float:
        t0 = time.perf_counter()
        if self.lt:
            self.orc.sample_block_lt(self.g, self.w, count, first, SEED)
        else:
            self.g.sample_block(count, first, SEED, self.threads)
        return time.perf_counter() - t0

    def describe(self, count: int, steps: int, first: int, seconds: float) -> dict:
        what = ("reference sample_block (oracle/_ref, unmodified sources, OpenMP)" if not self.lt else
                "C-restatement LT walk oc_sample_block_lt (the reference has no LT path)")
        return {"kind": self.kind, "cores": self.threads, "cpu_model": cpu_model(),
                "sample": f"{what}: {steps} x {count} RRR sets of the workload, global indices from {first}, "
                          f"{seconds:.1f} s; graph generated by oracle/gen_graph.c in {self.gen_s:.1f} s (untimed)"}


def run_reference_arm(args, cfg, rank, world):
    if rank != 0:
        return 0
    per_step = args.ref_samples or cfg["ref_samples"]
    rw = ReferenceWindow(cfg)
    idx = 0
    for _ in range(args.warmup):
        rw.sample(per_step, idx)
        idx += per_step
    first = idx
    t = 0.0
    for _ in range(args.steps):
        t += rw.sample(per_step, idx)
        idx += per_step
    value = per_step * args.steps / t
    cpu = {"value": value, "unit": "samples/s", **rw.describe(per_step, args.steps, first, t)}
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * t / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": DTYPE, "data": "synthetic",
        "config": config_dict(args, cfg, world),
        "step": f"one reference sample_block window of {per_step} RRR sets (sampling is ~99% of the reference "
                "IMM time on these configs, SURVEY.md §3.1; its full IMM re-samples the estimation sets, so "
                "this rate is an upper bound on the reference's theta / IMM-seconds)",
        "cpu_baseline": cpu,
        "e2e": {"value": value, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def config_dict(args, cfg, world):
    # identical in both arms (the driver compares them)
    return {"workload": args.config, "desc": cfg["desc"], "seed": SEED,
            "l2": "GPU arm: a 256 MB write flushes L2 (126 MB) between steps; the c4 and c5 graphs are also larger than L2",
            "parallelism": f"replicas x{world}"}


# ------------------------------------------------------------------ our arm
_PINNED = []

def pinned_copy(a: np.ndarray) -> np.ndarray:
    import torch

    t = torch.empty(a.size, dtype={np.dtype(np.uint64): torch.int64, np.dtype(np.uint32): torch.int32,
                                   np.dtype(np.float64): torch.float64}[a.dtype], pin_memory=True)
    v = t.numpy().view(a.dtype)
    v[:] = a
    _PINNED.append(t)  # keep the pinned buffer alive
    return v


def run_ours(args, cfg, rank, world, local):
    import torch

    import paper_2208_00613_b200 as im

    torch.cuda.set_device(local)
    dev = im.default_device(local)
    stream = torch.cuda.ExternalStream(dev.stream, device=f"cuda:{local}")
    transposed = bool(cfg.get("device_gen"))
    if transposed:
        # large configs: generated in HBM as the reverse CSR (identical to the host generator +
        # transpose, tests/test_gpu_parity.py); the e2e leg uploads that reverse CSR from host
        gen = cfg["gen"]
        dg = im.DeviceGraph.generate_rmat(gen[1], gen[2], 0.57, 0.19, 0.19, gen[3], weights=cfg["weights"][0],
                                          p=cfg["weights"][1], device=dev)
        off, tgt, _ = dg.download(probs=False)
    else:
        g = make_graph(im, cfg)
        off, tgt, pr, _ = g.arrays()
        dg = im.DeviceGraph.from_arrays(int(off.size - 1), off, tgt, pr, False, device=dev)
    n, m = int(off.size - 1), int(tgt.size)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device=f"cuda:{local}")  # > L2 (126 MB)
    run_kw = dict(epsilon=cfg["eps"], blocks=cfg["blocks"], mode=cfg["mode"], seed=SEED)
    if "lt_seed" in cfg:  # config 3: LT diffusion (extension; weights generated in HBM)
        dg.set_lt_random(cfg["lt_seed"])
        run_kw["model"] = 1

    def one_step():
        return im.run_device(dg, cfg["k"], **run_kw)

    tw = time.perf_counter()
    warm_ms = []  # wall time per warm-up step; the first runs on a graph the device has not seen
    for _ in range(args.warmup):
        with torch.cuda.stream(stream):
            flush.fill_(1)  # (warms the flush kernel too: its first launch loads the module, ~40 ms)
            torch.cuda.Event(enable_timing=True).record(stream)
        dev.synchronize()
        t1 = time.perf_counter()
        one_step()
        dev.synchronize()
        warm_ms.append(round((time.perf_counter() - t1) * 1e3, 2))
    dev.synchronize()
    # clocks polled once a second in regions >= 2 s, else right after the region (an
    # nvidia-smi query could stall the driver for tens of ms; NVML is polled in-process)
    expect_s = (time.perf_counter() - tw) / max(args.warmup, 1) * args.steps
    period_ms = int(os.environ.get("BENCH_CLOCK_MS", "0")) or (1000 if expect_s >= 2.0 else 2000)

    # ---- timed: graph resident in HBM ----
    dev.profile(True)
    dev.reset_stats()
    launches0 = dev.kernel_launches
    barrier(world)
    torch.cuda.synchronize()
    dev.synchronize()
    samples = 0
    results = []
    with clock_sampler(local, period_ms) as clk:
        clk.wait_first()
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            ev0.record(stream)
        marks = []
        for _ in range(args.steps):
            with torch.cuda.stream(stream):
                flush.fill_(1)  # L2 flush between steps, on the library stream
                e = torch.cuda.Event(enable_timing=True)
                e.record(stream)
                marks.append(e)
            r = one_step()
            samples += r["theta"]  # the sets the result uses (look-ahead may have drawn more)
            results.append(r)
        with torch.cuda.stream(stream):
            ev1.record(stream)
        ev1.synchronize()
        clk.ensure_one()
    dev.synchronize()
    torch.cuda.synchronize()
    barrier(world)
    ms_local = ev0.elapsed_time(ev1)
    # per step: from the end of its L2 flush to the next step's (or the region's end)
    step_ms = [marks[i].elapsed_time(marks[i + 1] if i + 1 < len(marks) else ev1) for i in range(len(marks))]
    launches = dev.kernel_launches - launches0
    samp = dev.kernel_stats("sample")
    hsel = dev.kernel_stats("hselect")
    enc = dev.kernel_stats("encode")
    dev.profile(False)

    ms = max_over_ranks(ms_local, world)
    total_samples = sum_over_ranks(samples, world)
    value = total_samples / (ms / 1000.0)

    # ---- e2e: from pinned host buffers through the C-ABI ----
    # the inputs are the CSR and the config's weight model: the probabilities are assigned on
    # the device (immx_graph_upload_model, assign_weights with float32 values), so only the
    # CSR crosses PCIe
    p_off, p_tgt = pinned_copy(off), pinned_copy(tgt)
    h2d = p_off.nbytes + p_tgt.nbytes
    d2h = cfg["k"] * (4 + 8 + 8) + 16 * 8 + 12 * 8 + cfg["blocks"] * 24
    barrier(world)
    dev.synchronize()
    t0 = time.perf_counter()
    e2e_samples = 0
    e2e_steps = args.steps
    for _ in range(e2e_steps):
        dge = im.DeviceGraph.from_arrays(n, p_off, p_tgt, None, transposed, device=dev, weights=cfg["weights"][0],
                                         p=cfg["weights"][1])
        if "lt_seed" in cfg:
            dge.set_lt_random(cfg["lt_seed"])
        r = im.run_device(dge, cfg["k"], **run_kw)  # results land in host memory
        e2e_samples += r["theta"]
        del dge
    dev.synchronize()
    e2e_s = max_over_ranks(time.perf_counter() - t0, world)
    e2e_value = sum_over_ranks(e2e_samples, world) / e2e_s

    if rank != 0:
        return 0
    r0 = results[-1]
    peak, peak_kind = load_peaks()
    samp_gbs = samp["bytes"] / (samp["ms"] / 1000.0) / 1e9 if samp["ms"] else None
    # DRAM bytes per launch: the dram/algorithmic ratio of the ncu --set full capture of the
    # same kernel on this config (profiles/), applied to this run's bytes per launch
    traffic = None
    issue = None
    prof = os.path.join(ROOT, "profiles", "ncu_sampler_traffic.json")
    clocks = clk.summary()
    if os.path.exists(prof):
        try:
            with open(prof) as f:
                pc = json.load(f)[args.config]
            traffic = pc["dram_over_alg"] * samp["bytes"] / max(samp["launches"], 1)
            # the sampler's real bound: instruction issue (ALU-heavy integer work on an
            # L2-resident graph).  warp-instructions per edge from the ncu capture x the live
            # edge rate of the kernel, against 4 issue slots per SM per clock
            edges = sum(x["edges_scanned"] for x in results)
            eps = edges / (samp["ms"] / 1000.0) if samp["ms"] else None
            sm_mhz = clocks.get("sm_mhz") or 1965.0
            if eps and pc.get("warp_inst_per_edge"):
                ach = eps * pc["warp_inst_per_edge"]
                pk = 4 * torch.cuda.get_device_properties(local).multi_processor_count * sm_mhz * 1e6
                issue = {"bound": "issue", "achieved": ach, "peak": pk, "unit": "warp-inst/s", "frac": ach / pk,
                         "warp_inst_per_edge": pc["warp_inst_per_edge"], "edges_per_s": eps,
                         "source": "profiles/ncu_sampler_traffic.json (ncu instruction count of the same kernel)"}
        except Exception:
            traffic = None

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        try:
            per = args.ref_samples or cfg["ref_samples"]
            rw = ReferenceWindow(cfg)
            dt = rw.sample(per, 0)
            cpu = {"value": per / dt, "unit": "samples/s", **rw.describe(per, 1, 0, dt)}
            del rw
        except Exception as ex:  # reference build missing on this box
            cpu = {"value": None, "unit": "samples/s", "cores": 0, "kind": "reference", "sample": f"unavailable: {ex}"}
    line = {
        "metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": DTYPE, "data": "synthetic",
        "config": config_dict(args, cfg, world),
        "theta": r0["theta"], "samples_drawn": r0["samples_drawn"], "reuse_pool": True,
        "scheduling_priors": "the timed steps run with the mean set size (arena sizing) and the covered fraction "
                             "(look-ahead sampling) the device remembered from the warm-up steps on this graph shape; "
                             "they choose launch sizes only, every result is the reference's (DESIGN.md section 2)",
        "imm_end_to_end_s": ms / args.steps / 1000.0,
        "step_ms": [round(x, 2) for x in step_ms],
        "warmup_step_ms": warm_ms,  # [0]: no scheduling priors yet (and one-time costs: module load, pool growth)
        "compression_ratio": r0["compression_ratio"],
        "dense_sets": r0.get("dense_sets", 0),
        "compression_ratio_device": r0["raw_bytes"] / r0["device_store_bytes"] if r0["device_store_bytes"] else None,
        "device_memory": {"peak_bytes": r0["device_peak_bytes"], "resident_after_run_bytes": r0["device_resident_bytes"],
                          "graph_bytes": r0["device_graph_bytes"], "store_bytes": r0["device_store_bytes"],
                          "ledger_peak_bytes": r0["peak_bytes"],
                          "note": "peak/resident = stream-ordered pool high-water / in-use bytes of the run (graph "
                                  "included); ledger = the reference's logical MemoryLedger peak"},
        "edges_examined_per_s": sum(x["edges_scanned"] for x in results) / (ms_local / 1000.0),
        "phase_seconds": r0["phase_seconds"],
        "seeds_head": r0["seeds"][:5],
        "roofline": {"bound": "hbm", "achieved": samp_gbs, "peak": peak, "unit": "GB/s",
                     "frac": (samp_gbs / peak) if samp_gbs else None, "traffic": traffic,
                     "kernel": "rrr_kernel (LT walks)" if "lt_seed" in cfg else "rrr_block_kernel (IC sampler)",
                     "peak_kind": peak_kind, "launches": samp["launches"],
                     "alg_bytes_per_launch": samp["bytes"] / max(samp["launches"], 1),
                     "avg_launch_ms": samp["ms"] / max(samp["launches"], 1)},
        "roofline_issue": issue,
        "select_roofline": {"achieved": hsel["bytes"] / (hsel["ms"] / 1000) / 1e9 if hsel["ms"] else None,
                            "unit": "GB/s", "launches": hsel["launches"], "ms": hsel["ms"]},
        "encode_roofline": {"achieved": enc["bytes"] / (enc["ms"] / 1000) / 1e9 if enc["ms"] else None,
                            "unit": "GB/s", "launches": enc["launches"], "ms": enc["ms"]},
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_value, "unit": "samples/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "steps": e2e_steps},
        "gpu_launches": launches,
        "clocks": clocks,
    }
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c5", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--ref-samples", type=int, default=0, help="reference window per step (default: per config)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3  # timing rule: at least 3 warm-up steps
    rank, world, local = dist_env()
    cfg = CONFIGS[args.config]
    if world > 1:
        import torch.distributed as dist

        if args.impl == "reference":
            dist.init_process_group("gloo")
        else:
            import torch

            torch.cuda.set_device(local)
            dist.init_process_group("nccl")
    try:
        if args.impl == "reference":
            rc = run_reference_arm(args, cfg, rank, world)
        else:
            rc = run_ours(args, cfg, rank, world, local)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()
    return rc


if __name__ == "__main__":
    sys.exit(main())
