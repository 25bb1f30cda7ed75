#!/usr/bin/env python
"""bench.py -- seconds per randomized-QLP factorisation on B200 (BASELINE.json metric).

One "step" = one whole factorisation (Ω, every A-pass, orthonormalisations, the CPQR/QLP
tail and the assembly of Q, T, P) of the workload's synthetic matrix, already resident in
HBM.  Default workload: BASELINE.json configs[1] ("c2": ERQLP fp64, m = n = 4096, k = 100,
p = 10, q = 1, d = 2).  Prints ONE JSON line (rank 0).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c1|c1e|c2|c3|c4|c5w]
  python bench.py --impl reference ...   # the CPU oracle (oracle/) timed on this host's cores
For N > 1 launch with torchrun (one rank per GPU, NCCL); A is row-sharded with the per-rank
row count of the workload fixed (weak scaling: global m = N x m_workload).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from synthetic import CONFIGS, make_A_config  # noqa: E402

FP64_DMMA_PEAK_TFLOPS = 37.07   # measured: tools/microbench/fp64_peak.cu on this pool (profiles/r01_fp64_peak.txt)
FP64_NOMINAL_TFLOPS = 37.2      # 148 SMs x 64 FP64 FMA/clk x 2 x 1.965 GHz
METRIC = "RQLP sec/factorization"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {}


def describe(c) -> dict:
    return {"workload": f"{c.name}: {c.variant.upper()} fp64 m={c.m} n={c.n} k={c.k} p={c.p} q={c.q}"
                        + (f" d={c.d}" if c.d else "") + (f" b={c.b}" if c.b else "")
                        + f" spectrum={c.spectrum}" + (f" rank={c.rank}" if c.rank else "")
                        + (f" noise={c.noise:g}" if c.noise else ""),
            "m": c.m, "n": c.n, "k": c.k, "p": c.p, "l": c.l, "q": c.q, "d": c.d, "b": c.b}


def passes(c) -> int:
    return 2 + 2 * c.q


class ClockSampler:
    """SM clock and clock-event (throttle) reasons sampled every ~2 ms by NVML in a background
    thread; the summary keeps the samples taken inside the timed region (the `with` block; the
    nearest later sample if the region is shorter than the period).  nvidia-smi is the fallback
    when NVML is unavailable."""

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"))
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []   # (t, sm_mhz, reasons)
        self.mx = None
        self.nv = None
        self.thread = None
        self.stop = False
        self.p = None
        self.out = ""

    def _nvml_handle(self):
        import pynvml
        pynvml.nvmlInit()
        try:
            bus = torch.cuda.get_device_properties(self.index).pci_bus_id
            dom = torch.cuda.get_device_properties(self.index).pci_domain_id
            dev = torch.cuda.get_device_properties(self.index).pci_device_id
            return pynvml, pynvml.nvmlDeviceGetHandleByPciBusId(f"{dom:08x}:{bus:02x}:{dev:02x}.0")
        except Exception:
            return pynvml, pynvml.nvmlDeviceGetHandleByIndex(self.index)

    def _loop(self, nv, h):
        while not self.stop:
            try:
                sm = float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
                bits = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                rs = [nm for nm, attr in self.REASONS if bits & getattr(nv, attr, 0)]
                self.samples.append((time.perf_counter(), sm, rs))
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        try:
            import threading
            nv, h = self._nvml_handle()
            self.nv = nv
            self.mx = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
            self.thread = threading.Thread(target=self._loop, args=(nv, h), daemon=True)
            self.thread.start()
            while not self.samples:
                time.sleep(0.001)
        except Exception:
            self.nv = None
            try:
                self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                           "--format=csv,noheader,nounits", "-lms", "100"],
                                          stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            except Exception:
                self.p = None
        self.t0 = time.perf_counter()
        return self

    def __exit__(self, *exc):
        self.t1 = time.perf_counter()
        if self.thread is not None:
            while not any(t >= self.t0 for t, _, _ in self.samples):
                time.sleep(0.001)
            self.stop = True
            self.thread.join(timeout=1)
        if self.p is not None:
            time.sleep(0.25)
            self.p.terminate()
            try:
                self.out, _ = self.p.communicate(timeout=5)
            except Exception:
                self.p.kill()
        return False

    def summary(self) -> dict:
        if self.nv is not None:
            inside = [s for s in self.samples if self.t0 <= s[0] <= self.t1]
            if not inside:
                inside = [min((s for s in self.samples if s[0] >= self.t0), key=lambda s: s[0])]
            reasons = sorted({r for _, _, rs in inside for r in rs})
            return {"sm_mhz": statistics.median(s[1] for s in inside), "sm_max_mhz": self.mx,
                    "reasons": reasons, "samples": len(inside), "source": "nvml"}
        sms, mx, reasons = [], None, set()
        names = [nm for nm, _ in self.REASONS]
        for line in (self.out or "").splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 6:
                continue
            try:
                sms.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for nm, v in zip(names, f[2:6]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sms) if sms else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sms), "source": "nvidia-smi"}


def flush_l2(buf: torch.Tensor):
    buf.add_(1.0)   # 256 MB write > 126 MB L2


def load_traffic(name: str):
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            return json.load(f).get(name)
    except Exception:
        return None


# ---------------------------------------------------------------------------- oracle arm
def oracle_time(A_np, c, budget_s: float = 12.0):
    """Time the CPU oracle (as it stands) on a bounded sample of workload c.  Returns
    (sec_per_factorisation_estimate, sample description, threads)."""
    import oracle
    oracle.build()
    m = A_np.shape[0]
    full_work = passes(c) * 2.0 * c.m * c.n * c.l
    # sample: the first m_s rows of A (same n, k, p, q, d, b) -- the A-passes scale with m, the
    # tail does not, so sec(full) ~= sec(sample) * m / m_s is an upper-bound-leaning estimate.
    gflops_guess = 15.0 * oracle.num_threads() / 8
    m_s = m
    if full_work / (gflops_guess * 1e9) > budget_s:
        m_s = max(c.l + 1, int(m * budget_s * gflops_guess * 1e9 / full_work))
        m_s = min(m, m_s)
    As = A_np[:m_s]
    reps, t_tot = 0, 0.0
    while True:
        t0 = time.perf_counter()
        if c.b is not None:
            oracle.brqlp(As, c.k, c.p, b=c.b, q=c.q, seed=c.seed)
        else:
            oracle.rqlp(As, c.k, c.p, q=c.q, d=c.d, seed=c.seed)
        t_tot += time.perf_counter() - t0
        reps += 1
        if t_tot >= budget_s * 0.5 or reps >= 5:
            break
    sec = t_tot / reps * (m / m_s)
    sample = (f"{reps} oracle factorisation(s) of the first {m_s} of {m} rows (n={c.n}, l={c.l}, q={c.q}, d={c.d}"
              + (f", b={c.b}" if c.b else "") + ")" + (f", scaled by m/m_s={m / m_s:.2f}" if m_s < m else ""))
    return sec, sample, oracle.num_threads()


def run_reference(args, c):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    torch.manual_seed(0)
    A = make_A_config(c, device="cpu")
    A_np = A.numpy()  # column-major view (m, n)
    import oracle
    oracle.build()
    secs = []
    for i in range(args.warmup + args.steps):
        s, sample, th = oracle_time(A_np, c, budget_s=6.0)
        if i >= args.warmup:
            secs.append(s)
    val = sum(secs) / len(secs)
    line = {"metric": METRIC, "value": val, "unit": "s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": val * 1e3, "higher_is_better": False, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": describe(c),
            "cpu_baseline": {"value": val, "unit": "s", "cores": th, "kind": "oracle", "sample": sample},
            "e2e": {"value": val, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------- GPU arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    c = CONFIGS[args.workload]
    if args.impl == "reference":
        return run_reference(args, c)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    group = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
        group = dist.group.WORLD

    import paper_1811_09334_b200 as rq
    from paper_1811_09334_b200 import build as rqbuild
    rqbuild.build()

    # A: per-rank row block of the weak-scaled matrix (global m = world * c.m)
    import dataclasses

    from paper_1811_09334_b200.dist import max_over_ranks, row_block
    cg = dataclasses.replace(c, m=c.m * world)
    r0, r1 = row_block(cg.m, rank, world)
    t0 = time.time()
    A = make_A_config(cg, device=dev, row_range=(r0, r1) if world > 1 else None)
    torch.cuda.synchronize()
    log(f"[bench] rank {rank}: A {tuple(A.shape)} generated in {time.time() - t0:.1f}s")
    handle = rq.Handle(device=dev, group=group)
    handle.set_timing(True)
    flushbuf = torch.zeros(32 * 1024 * 1024, dtype=torch.float64, device=dev)
    stream = handle.stream

    def step():
        return rq.factorize(A, c.k, c.p, q=c.q, d=c.d, b=c.b, seed=c.seed, handle=handle)

    def barrier():
        if group is not None:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    out = None
    for _ in range(args.warmup):
        out = None   # release the previous outputs first: the next call then gets the same buffers,
        out = step()  # i.e. the same graph-cache key (eager, capture, then replays)
        flush_l2(flushbuf)
    barrier()

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    stage_ms: dict[str, list[float]] = {}
    launches = 0
    with ClockSampler(local) as clk:
        barrier()
        for i in range(args.steps):
            flush_l2(flushbuf)
            out = None
            ev[i][0].record(stream)
            out = step()
            ev[i][1].record(stream)
            launches += handle.launches()
        barrier()
    # No host synchronisation inside the timed loop: the host enqueues step i+1 while the device
    # runs step i, so the per-step event pairs measure device time (the host's per-call cost is
    # in the e2e number).  The stage events are those of the last timed step.
    for name, ms in handle.timing():
        stage_ms.setdefault(name, []).append(ms)
    stage_steps = 1
    step_ms = [a.elapsed_time(b) for a, b in ev]
    total_ms = max_over_ranks(sum(step_ms), group, dev)
    ms_per_step = total_ms / args.steps
    flags = handle.sync()

    # ---- A-pass roofline (the hot path: 92-97% of the flops): algorithmic A-pass flops per step
    # (passes x 2 m n l; BRQLP: the width-l sketch + (2q+1) width-b_j passes per block, same
    # total) / the summed per-pass CUDA-event durations inside the timed region.
    pass_names = [k for k in stage_ms if k.startswith("pass_")]
    pass_times = [t for k in pass_names for t in stage_ms[k]]
    flops_pass = 2.0 * c.m * c.n * c.l
    bytes_pass = 8.0 * (c.m * c.n + c.m * c.l + c.n * c.l)
    roof = None
    if pass_times:
        mean_pass_ms = sum(pass_times) / stage_steps / passes(c)   # per width-l-equivalent pass
        ach = flops_pass / (mean_pass_ms * 1e-3) / 1e12
        roof = {"bound": "tensor", "achieved": round(ach, 3), "peak": FP64_DMMA_PEAK_TFLOPS, "unit": "TFLOP/s",
                "frac": round(ach / FP64_DMMA_PEAK_TFLOPS, 4), "traffic": load_traffic(c.name),
                "kernel": "A-pass: FP64 DMMA GEMM gemm_tma_kernel (Y=AX and B=V^T A / A^T V, incl. split-K "
                          "reduce); achieved = algorithmic A-pass flops / summed pass event time",
                "algorithmic_flops_per_launch": flops_pass, "algorithmic_bytes_per_launch": bytes_pass,
                "mean_pass_ms": round(mean_pass_ms, 4),
                "peak_source": "measured DMMA m8n8k4 FP64 microbenchmark (tools/microbench/fp64_peak.cu, "
                               "profiles/r01_fp64_peak.txt); MEASURED_PEAKS.json has no FP64 entry",
                "hbm_frac": round(bytes_pass / (mean_pass_ms * 1e-3) / 1e9 / measured_peaks().get("hbm_gbs", 6540.8),
                                  4)}
    apass_total_ms = sum(pass_times) / stage_steps if pass_times else None

    # ---- e2e through the public API with HOST buffers (pinned)
    e2e = None
    if not args.no_e2e and world == 1:
        A_h = torch.empty(c.n, c.m, dtype=torch.float64, pin_memory=True).t()
        A_h.copy_(A)
        l = c.l
        outs = tuple(torch.empty(cc, r, dtype=torch.float64, pin_memory=True).t()
                     for r, cc in ((c.m, l), (l, l), (c.n, l)))
        hh = rq.Handle(device=dev)
        for _ in range(2):
            rq.factorize_host(A_h, c.k, c.p, q=c.q, d=c.d, b=c.b, seed=c.seed, handle=hh, out=outs)
        ts = []
        for _ in range(max(3, min(args.steps, 10))):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            rq.factorize_host(A_h, c.k, c.p, q=c.q, d=c.d, b=c.b, seed=c.seed, handle=hh, out=outs)
            ts.append(time.perf_counter() - t0)
        e2e = {"value": sum(ts) / len(ts), "unit": "s", "h2d_bytes_per_step": 8 * c.m * c.n,
               "d2h_bytes_per_step": 8 * (c.m * l + l * l + c.n * l), "api": "rqlp_factorize (C ABI, pinned host)"}
        del hh

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        A_np = A.cpu().numpy()
        sec, sample, th = oracle_time(A_np, c)
        cpu = {"value": sec, "unit": "s", "cores": th, "kind": "oracle", "sample": sample}

    if rank == 0:
        line = {"metric": METRIC, "value": ms_per_step / 1e3, "unit": "s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": False, "scaling": "weak",
                "vs_baseline": None, "dtype": "f64",
                "data": "synthetic: A = U diag(sigma) V^T (+noise), Haar U, V from torch.linalg.qr of seeded "
                        "Gaussians; Omega from Philox4x64-10 (DESIGN.md §4)",
                "config": {**describe(c), "global_m": cg.m, "parallelism": f"rows sharded over {world} rank(s)",
                           "l2": "flushed between timed steps (256 MB write, untimed)",
                           "apass_ms_per_step": apass_total_ms},
                "apass_tflops": (passes(c) * flops_pass / (apass_total_ms * 1e-3) / 1e12) if apass_total_ms else None,
                "tflops_effective": passes(c) * 2.0 * cg.m * c.n * c.l / (ms_per_step * 1e-3) / 1e12,
                "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": launches, "clocks": clk.summary(), "step_ms": [round(t, 4) for t in step_ms],
                "stages_ms": {k: round(sum(v) / len(v), 4) for k, v in stage_ms.items()},
                "device_flags": flags}
        print(json.dumps(line), flush=True)
    if group is not None:
        torch.distributed.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
