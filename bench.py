#!/usr/bin/env python
"""bench.py -- seconds per randomized-QLP factorisation on B200 (BASELINE.json metric).

One "step" = one whole factorisation (Ω, every A-pass, orthonormalisations, the CPQR/QLP
tail and the assembly of Q, T, P) of the workload's synthetic matrix, already resident in
HBM.  Default workload: BASELINE.json configs[3] ("c4": Block RQLP fp64, m = 262144,
n = 16384, k = 512, p = 16, b = 64, q = 1) -- the configuration the metric is quoted on at
1/2/4/8 B200 and the largest one that fits one GPU.  Prints ONE JSON line (rank 0).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c1|c1e|c2|c3|c4|c5|c5w]
                  [--scaling strong|weak]
  python bench.py --impl reference ...   # the CPU oracle (oracle/) timed on this host's cores
For N > 1 launch with torchrun (one rank per GPU, NCCL).  A is row-sharded.  --scaling strong
(default for c4 and c5, BASELINE's 1/2/4/8-GPU configs) keeps the global m of the workload and
gives each rank ~m/N rows; --scaling weak (default for c5w) keeps m rows per rank (global m =
N x m).
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
METRIC = "RQLP sec/factorization; A-pass TFLOP/s as % roofline at 1/2/4/8 B200"


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
                try:
                    pw = nv.nvmlDeviceGetPowerUsage(h) / 1000.0
                except Exception:
                    pw = None
                self.samples.append((time.perf_counter(), sm, rs, pw))
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
            while not any(s[0] >= self.t0 for s in self.samples):
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
            reasons = sorted({r for s in inside for r in s[2]})
            mhz = sorted(s[1] for s in inside)
            pws = [s[3] for s in inside if s[3] is not None]
            return {"sm_mhz": statistics.median(mhz), "sm_max_mhz": self.mx,
                    "reasons": reasons, "samples": len(inside), "source": "nvml",
                    "sm_mhz_min": mhz[0], "sm_mhz_p05": mhz[len(mhz) // 20],
                    "power_cap_sample_frac": round(sum(1 for s in inside if "sw_power_cap" in s[2]) / len(inside), 4),
                    "power_w_mean": round(sum(pws) / len(pws), 1) if pws else None,
                    "power_w_max": round(max(pws), 1) if pws else None}
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
def _oracle_run(A_np, c):
    import oracle
    if c.b is not None:
        oracle.brqlp(A_np, c.k, c.p, b=c.b, q=c.q, seed=c.seed)
    else:
        oracle.rqlp(A_np, c.k, c.p, q=c.q, d=c.d, seed=c.seed)


def sample_rows(c, budget_s: float, threads: int) -> int:
    """Rows of the bounded oracle sample: the A-passes scale with m (the tail does not), so the
    first m_s rows with the same n, k, p, q, d, b cost ~ m_s/m of the whole factorisation."""
    full_work = passes(c) * 2.0 * c.m * c.n * c.l
    gflops_guess = 15.0 * threads / 8
    m_s = c.m
    if full_work / (gflops_guess * 1e9) > budget_s:
        m_s = max(c.l + 1, int(c.m * budget_s * gflops_guess * 1e9 / full_work))
    return min(c.m, m_s)


def oracle_time(A_rows, c, budget_s: float = 12.0, reps_max: int = 5):
    """Time the CPU oracle (as it stands) on a bounded sample of workload c.  `A_rows(m_s)` returns
    the first m_s rows of A as a column-major numpy array.  Returns (sec_per_factorisation_estimate,
    sample description, threads)."""
    import oracle
    oracle.build()
    th = oracle.num_threads()
    m_s = sample_rows(c, budget_s, th)
    As = A_rows(m_s)
    reps, t_tot = 0, 0.0
    while True:
        t0 = time.perf_counter()
        _oracle_run(As, c)
        t_tot += time.perf_counter() - t0
        reps += 1
        if t_tot >= budget_s * 0.5 or reps >= reps_max:
            break
    sec = t_tot / reps * (c.m / m_s)
    sample = (f"{reps} oracle factorisation(s) of the first {m_s} of {c.m} rows (n={c.n}, l={c.l}, q={c.q}, d={c.d}"
              + (f", b={c.b}" if c.b else "") + ")" + (f", scaled by m/m_s={c.m / m_s:.2f}" if m_s < c.m else ""))
    return sec, sample, th


def single_thread_times() -> dict:
    """The oracle on ONE host thread at C1 (whole factorisation) and C2 (whole factorisation,
    one run): SURVEY §8(d)'s single-thread CPU figures."""
    import oracle
    from synthetic import CONFIGS as C
    out = {}
    prev = oracle.num_threads()
    oracle.set_num_threads(1)
    try:
        for name in ("c1", "c2"):
            c = C[name]
            A = make_A_config(c, device="cuda" if torch.cuda.is_available() else "cpu").cpu().numpy()
            t0 = time.perf_counter()
            _oracle_run(A, c)
            out[name] = round(time.perf_counter() - t0, 4)
    finally:
        oracle.set_num_threads(prev)
    return out


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def config_dict(c, world: int, scaling: str, m_global: int) -> dict:
    """The `config` object of the JSON line -- identical for both arms."""
    return {**describe(c), "global_m": m_global, "scaling": scaling,
            "parallelism": f"rows of A sharded over {world} rank(s) ({scaling} scaling)",
            "l2": "flushed between timed steps (256 MB write, untimed); A alone is larger than L2"}


def resolve(args):
    c = CONFIGS[args.workload]
    scaling = args.scaling or ("weak" if c.name == "c5w" else "strong")
    return c, scaling


def run_reference(args, c, scaling):
    """--impl reference: the CPU oracle as it stands on the host cores, on a bounded row sample of
    the workload (rank 0 only; other ranks exit without work)."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return 0
    import dataclasses
    import oracle
    oracle.build()
    cg = dataclasses.replace(c, m=c.m * world) if scaling == "weak" else c
    th = oracle.num_threads()
    m_s = sample_rows(cg, 5.0, th)
    dev = "cuda" if torch.cuda.is_available() else "cpu"   # data generation only (torch), not the method
    A_s = make_A_config(cg, device=dev, row_range=(0, m_s)).cpu().numpy()
    if dev == "cuda":
        torch.cuda.empty_cache()
    secs = []
    sample = ""
    for i in range(args.warmup + args.steps):
        s, sample, th = oracle_time(lambda ms: A_s[:ms], cg, budget_s=5.0, reps_max=1)
        if i >= args.warmup:
            secs.append(s)
    val = sum(secs) / len(secs)
    line = {"metric": METRIC, "value": val, "unit": "s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": val * 1e3, "higher_is_better": False, "scaling": scaling,
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": config_dict(c, world, scaling, cg.m),
            "cpu_baseline": {"value": val, "unit": "s", "cores": th, "kind": "oracle", "sample": sample,
                             "cpu_model": cpu_model()},
            "e2e": {"value": val, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------- GPU arm
E2E_HOST_LIMIT_BYTES = 96e9
DEFAULT_STEPS = {"c1": (20, 5), "c1e": (20, 5), "c2": (20, 5), "c3": (10, 3), "c4": (5, 3), "c5": (3, 3),
                 "c5w": (3, 3)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None)
    ap.add_argument("--warmup", type=int, default=None)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c4", choices=sorted(CONFIGS))
    ap.add_argument("--scaling", default=None, choices=["strong", "weak"])
    ap.add_argument("--shard-of", type=int, default=0,
                    help="diagnostic (1 GPU): time ONE rank's row block of an N-GPU strong-scaling run through the "
                         "row-sharded NCCL handle (a world-size-1 communicator: every exchange step is issued, "
                         "no link time) -- the per-rank compute time behind the projected efficiency in DESIGN.md")
    ap.add_argument("--shard-plain", action="store_true",
                    help="with --shard-of: the same row block on the single-GPU handle (graph replay, no exchange "
                         "steps) -- separates the sharded path's own overhead from the smaller shape's efficiency")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    ds, dw = DEFAULT_STEPS.get(args.workload, (5, 3))
    args.steps = ds if args.steps is None else args.steps
    args.warmup = max(dw if args.warmup is None else args.warmup, 3)
    c, scaling = resolve(args)
    if args.impl == "reference":
        return run_reference(args, c, scaling)

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
    elif args.shard_of > 1 and args.shard_plain:
        args.no_cpu_baseline = True
    elif args.shard_of > 1:
        import socket

        import torch.distributed as dist
        sk = socket.socket()
        sk.bind(("127.0.0.1", 0))
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(sk.getsockname()[1]))
        sk.close()
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
        group = dist.group.WORLD
        args.no_cpu_baseline = True

    import paper_1811_09334_b200 as rq
    from paper_1811_09334_b200 import build as rqbuild
    rqbuild.build()

    import dataclasses

    from paper_1811_09334_b200.dist import max_over_ranks, row_block
    cg = dataclasses.replace(c, m=c.m * world) if scaling == "weak" else c
    r0, r1 = row_block(cg.m, rank, world)
    if args.shard_of > 1:   # rank 0's block of an N-rank run
        r0, r1 = row_block(cg.m, 0, args.shard_of)
    m_loc = r1 - r0
    t0 = time.time()
    A = make_A_config(cg, device=dev, row_range=(r0, r1) if (world > 1 or args.shard_of > 1) else None)
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    log(f"[bench] rank {rank}: A {tuple(A.shape)} (rows {r0}..{r1} of {cg.m}) generated in {time.time() - t0:.1f}s")
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
    if world > 1:   # the replicated outputs (L, P, pivots) must be bit-identical on every rank
        chk = torch.stack([out["T"].contiguous().view(torch.int64).sum(), out["P"].contiguous().view(torch.int64).sum(),
                           out["piv0"].sum()])
        allc = [torch.zeros_like(chk) for _ in range(world)]
        torch.distributed.all_gather(allc, chk)
        replicated_identical = all(torch.equal(allc[0], x) for x in allc)
    else:
        replicated_identical = True

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
    timing_list = handle.timing()
    for name, ms in timing_list:
        stage_ms.setdefault(name, []).append(ms)
    step_ms = [a.elapsed_time(b) for a, b in ev]
    total_ms = max_over_ranks(sum(step_ms), group, dev)
    ms_per_step = total_ms / args.steps
    flags = handle.sync()

    # ---- A-pass roofline.  All A-passes together (92-97% of the flops): algorithmic A-pass flops per
    # width-l-equivalent pass on this rank (2 m_loc n l; BRQLP: the width-l sketch + (2q+1)
    # width-b_j passes per block, the same total) / the mean per-pass CUDA-event duration inside the
    # timed region (stage events of the last timed step, on the library's stream); max over ranks.
    pass_names = [k for k in stage_ms if k.startswith("pass_")]
    pass_ms_loc = sum(t for k in pass_names for t in stage_ms[k])
    pass_ms = max_over_ranks(pass_ms_loc, group, dev) if pass_names else 0.0
    flops_pass = 2.0 * m_loc * c.n * c.l
    bytes_pass = 8.0 * (m_loc * c.n + m_loc * c.l + c.n * c.l)
    apass = None
    if pass_ms > 0:
        mean_pass_ms = pass_ms / passes(c)
        apass = {"tflops_per_gpu": round(flops_pass / (mean_pass_ms * 1e-3) / 1e12, 3),
                 "mean_width_l_pass_ms": round(mean_pass_ms, 4), "apass_ms_per_step": round(pass_ms, 4)}
    # The dominant kernel's roofline: RQLP/ERQLP -- the width-l pass kernel (every A-pass);
    # BRQLP -- the width-b block pass (gemm_tma_kernel<b, TN>: A^(j-1)^T V_j and V_j^T A, 2 of the 3
    # passes of each full block, ~46 % of C4's step), its mean CUDA-event duration over the full
    # blocks of the last timed step.
    roof = None
    if c.b is not None:
        h_full = c.l // c.b
        tn = [ms for nm, ms in timing_list if nm in ("pass_block_AtV", "pass_block_project")]
        full = []    # per full block: q A^T V passes, 1 V^T A pass (q = 0 batches B = V^T A: none)
        for nm, per in (("pass_block_AtV", c.q), ("pass_block_project", 1)):
            xs = [ms for n2, ms in timing_list if n2 == nm]
            full += xs[:h_full * per]
        if full:
            kms = max_over_ranks(sum(full) / len(full), group, dev)
            kflops = 2.0 * m_loc * c.n * c.b
            kbytes = 8.0 * (m_loc * c.n + m_loc * c.b + c.n * c.b)
            ach = kflops / (kms * 1e-3) / 1e12
            roof = {"bound": "tensor", "achieved": round(ach, 3), "peak": FP64_DMMA_PEAK_TFLOPS, "unit": "TFLOP/s",
                    "frac": round(ach / FP64_DMMA_PEAK_TFLOPS, 4),
                    "traffic": load_traffic(c.name) if world == 1 else None,
                    "kernel": f"gemm_tma_kernel<{c.b}, TN>: the width-b BRQLP block pass (Z = A^T V_j, B_j = V_j^T A), "
                              "incl. its split-K reduce; mean CUDA-event time over the full blocks",
                    "algorithmic_flops_per_launch": kflops, "algorithmic_bytes_per_launch": kbytes,
                    "mean_launch_ms": round(kms, 4), "launches_per_step": len(full) + (len(tn) - len(full))}
    if roof is None and apass:
        ach = apass["tflops_per_gpu"]
        roof = {"bound": "tensor", "achieved": ach, "peak": FP64_DMMA_PEAK_TFLOPS, "unit": "TFLOP/s",
                "frac": round(ach / FP64_DMMA_PEAK_TFLOPS, 4), "traffic": load_traffic(c.name) if world == 1 else None,
                "kernel": "gemm_tma_kernel: the width-l A-pass (Y = A X, B = V^T A / A^T V), incl. its split-K reduce; "
                          "mean CUDA-event time per pass",
                "algorithmic_flops_per_launch": flops_pass, "algorithmic_bytes_per_launch": bytes_pass,
                "mean_launch_ms": apass["mean_width_l_pass_ms"]}
    if roof:
        roof["peak_source"] = ("measured DMMA m8n8k4 FP64 microbenchmark (tools/microbench/fp64_peak.cu, "
                               "profiles/r01_fp64_peak.txt); MEASURED_PEAKS.json has no FP64 entry")
        roof["hbm_frac"] = round(roof["algorithmic_bytes_per_launch"] / (roof["mean_launch_ms"] * 1e-3) / 1e9
                                 / measured_peaks().get("hbm_gbs", 6540.8), 4)
    # whole factorisation: the algorithmic A-pass flops of the step (the roofline-defining work)
    # over the step time, against the N-GPU FP64 peak (BASELINE's "slower of bytes@8TB/s and flops@peak")
    whole_flops = passes(c) * 2.0 * cg.m * c.n * c.l
    t_roof_flop = whole_flops / (world * FP64_DMMA_PEAK_TFLOPS * 1e12)
    t_roof_byte = passes(c) * 8.0 * (cg.m * c.n + cg.m * c.l + world * c.n * c.l) / (world * 8e12)
    whole = {"flops": whole_flops, "t_roof_s": max(t_roof_flop, t_roof_byte), "bound": "tensor" if t_roof_flop >= t_roof_byte else "hbm",
             "tflops": round(whole_flops / (ms_per_step * 1e-3) / 1e12, 3),
             "frac": round(max(t_roof_flop, t_roof_byte) / (ms_per_step * 1e-3), 4)}

    # ---- e2e through the public API with HOST buffers (pinned): rqlp_factorize copies this rank's
    # rows of A host->device, factorises and copies Q, T, P back, all inside the timed call
    e2e = None
    host_bytes = 8 * (m_loc * c.n + m_loc * c.l + c.l * c.l + c.n * c.l)
    if not args.no_e2e and host_bytes > E2E_HOST_LIMIT_BYTES:
        # the pinned host copy of this rank's rows would not fit comfortably in host memory (C5 whole on
        # one GPU: 137 GB of the box's 196 GB); no end-to-end number rather than a swapping one
        log(f"[bench] e2e skipped: {host_bytes / 1e9:.0f} GB of pinned host buffers > {E2E_HOST_LIMIT_BYTES / 1e9:.0f} GB")
        args.no_e2e = True
    if not args.no_e2e:
        l = c.l
        A_h = torch.empty(c.n, m_loc, dtype=torch.float64, pin_memory=True).t()
        A_h.copy_(A)
        outs = tuple(torch.empty(cc, r, dtype=torch.float64, pin_memory=True).t()
                     for r, cc in ((m_loc, l), (l, l), (c.n, l)))
        del A, out
        torch.cuda.empty_cache()
        hh = rq.Handle(device=dev, group=group)
        for _ in range(2):
            rq.factorize_host(A_h, c.k, c.p, q=c.q, d=c.d, b=c.b, seed=c.seed, handle=hh, out=outs)
        ts = []
        for _ in range(max(3, min(args.steps, 5))):
            barrier()
            t0 = time.perf_counter()
            rq.factorize_host(A_h, c.k, c.p, q=c.q, d=c.d, b=c.b, seed=c.seed, handle=hh, out=outs)
            ts.append(time.perf_counter() - t0)
        e2e_s = max_over_ranks(sum(ts) / len(ts), group, dev)
        e2e = {"value": e2e_s, "unit": "s", "h2d_bytes_per_step": 8 * cg.m * c.n,
               "d2h_bytes_per_step": 8 * (cg.m * l + world * (l * l + c.n * l)),
               "api": "rqlp_factorize (C ABI, pinned host buffers; max over ranks of the per-rank wall time)"}
        del hh

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        def rows(ms):
            return make_A_config(c, device=dev, row_range=(0, ms)).cpu().numpy()

        sec, sample, th = oracle_time(rows, c)
        cpu = {"value": sec, "unit": "s", "cores": th, "kind": "oracle", "sample": sample, "cpu_model": cpu_model(),
               "single_thread_s": single_thread_times()}

    if rank == 0:
        line = {"metric": METRIC, "value": ms_per_step / 1e3, "unit": "s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": False, "scaling": scaling,
                "vs_baseline": None, "dtype": "f64",
                "data": "synthetic: A = U diag(sigma) V^T (+noise), Haar U, V from torch.linalg.qr of seeded "
                        "Gaussians; Omega from Philox4x64-10 (DESIGN.md §4)",
                "config": config_dict(c, world, scaling, cg.m),
                "apass": apass,
                "tflops_effective": whole["tflops"],
                "roofline": roof, "roofline_whole_factorisation": whole, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": launches, "clocks": clk.summary(), "step_ms": [round(t, 4) for t in step_ms],
                "stages_ms": {k: round(sum(v) / len(v), 4) for k, v in stage_ms.items()},
                "stages_total_ms": {k: round(sum(v), 4) for k, v in stage_ms.items()},
                "replicated_outputs_identical": replicated_identical, "device_flags": flags}
        if args.shard_of > 1:
            line["shard_of"] = {"n_ranks": args.shard_of, "rows": m_loc, "handle": "single-GPU" if args.shard_plain else "nccl world 1",
                                "note": "ONE rank's block through the sharded (NCCL, world-size-1) handle; a "
                                        "diagnostic, not a bench value: roofline_whole_factorisation is meaningless here"}
        print(json.dumps(line), flush=True)
    if group is not None:
        torch.distributed.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
