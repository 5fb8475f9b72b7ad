#!/usr/bin/env python3
"""bench.py -- quartic-K3 quasi-F-split heights/sec on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--p 5] [--batch 100000] [--impl reference]

A "step" is one pass of the hot path (qfs_heights: power chain -> Witt carry -> operator matrix ->
matvec chain with early exit) over one batch of seeded synthetic quartics, generated with the
reference's sampler recipe (numpy default_rng([seed, worker]), one integers(0,p,35) draw per
surface, zero draws redrawn; search.py:92-98,103).  Default workload = BASELINE.json configs[1]:
100k random quartics over F_5 on one B200; the F_7 100k batch (configs[2]) is measured in the same
run and reported under "also".

One JSON line on stdout (rank 0).  `value` = whole-job surfaces/s with inputs resident in HBM;
`e2e` = the same through the public API with pinned HOST buffers (H2D/D2H inside the timed region);
`roofline` = the dominant kernel against the measured HBM peak; `cpu_baseline` = the C oracle
(oracle/, a port of the reference's CPU algorithm) on this box's host cores.
`--impl reference` times that CPU port alone (the reference itself is pure Python under
/root/reference and cannot travel to the GPU box).
"""
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

# surfaces/s that take the full operator path: F_5, F_7 on a 2080 Ti; F_11: one surface per 39-40 s on an RTX 3090
PAPER_RATE = {5: 1400.0, 7: 180.0, 11: 1.0 / 39.5}
PAPER_NOTE = {5: "~1400/s on a 2080 Ti", 7: "~180/s on a 2080 Ti", 11: "one surface per 39-40 s (0.025/s) on an RTX 3090"}


def reference_python_rate(p):
    """Rate of the UNMODIFIED reference (qfsplit, numpy + numba) measured in the authoring container (tools/measure_reference.py):
    it does not travel to the GPU box, so the box-side CPU arm is its C port and this is quoted beside it."""
    try:
        with open(os.path.join(ROOT, "profiles", "reference_python_rate.json")) as fh:
            j = json.load(fh)
        e = j[f"F_{p}"]
        return {"surfaces_per_s": e["surfaces_per_s"], "surfaces_per_s_per_core": e["surfaces_per_s_per_core"], "cores": j["cores"],
                "samples": e["samples"], "where": "authoring container, profiles/reference_python_rate.json"}
    except Exception:
        return None


def workload_name(p, batch):
    N, _ = SHAPES[p]
    return f"{batch} seeded random quartics over F_{p} per GPU ({N}x{N} operator), bound 10"
SHAPES = {3: (165, 2925), 5: (969, 91881), 7: (2925, 818805), 11: (12341, 14391741)}  # N, L


def sample_block(p, count, seed, worker):
    """`count` coefficient vectors exactly as search._worker_block draws them (search.py:103,92-98)."""
    from paper_2502_12428_b200.search import sample_block as sb
    return sb(p, count, seed, worker)


def cached_block(p, count, seed, worker):
    d = os.path.join(ROOT, "bench_cache")
    path = os.path.join(d, f"coeffs_p{p}_s{seed}_w{worker}_{count}.npy")
    try:
        if os.path.exists(path):
            return np.load(path)
    except Exception:
        pass
    c = sample_block(p, count, seed, worker)
    try:
        os.makedirs(d, exist_ok=True)
        np.save(path, c)
    except Exception:
        pass
    return c


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            j = json.load(fh)
        return float(j["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (measured copy bandwidth)"
    except Exception:
        return 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"


def measured_traffic(p, kernel, hard, launches):
    """dram__bytes_read.sum + dram__bytes_write.sum of `kernel` per launch from the committed `ncu --set full` capture
    (profiles/traffic.json).  The capture of the headline configuration is taken AT the benchmark's launch size (its `hard`
    equals this run's surfaces per launch: the number is the measured one); otherwise it is the capture's bytes per hard surface
    times this run's surfaces per launch.  None if no capture is on file."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            t = json.load(fh)
        e = t[f"p{p}"][kernel]
        per_launch = hard / launches
        if abs(e.get("hard_surfaces_in_capture", 0) - per_launch) <= 0.001 * per_launch:
            return e["dram_bytes_per_launch"]
        return e["dram_bytes_per_hard_surface"] * per_launch
    except Exception:
        return None


_SAMPLER_SRC = r"""
import sys, time
import pynvml as n
n.nvmlInit()
uuid = sys.argv[1]
try:
    h = n.nvmlDeviceGetHandleByUUID(uuid.encode()) if uuid != "-" else n.nvmlDeviceGetHandleByIndex(int(sys.argv[2]))
except Exception:
    h = n.nvmlDeviceGetHandleByIndex(int(sys.argv[2]))
get = getattr(n, "nvmlDeviceGetCurrentClocksEventReasons", None) or n.nvmlDeviceGetCurrentClocksThrottleReasons
print("max", n.nvmlDeviceGetMaxClockInfo(h, n.NVML_CLOCK_SM), flush=True)
while True:
    print(time.time(), n.nvmlDeviceGetClockInfo(h, n.NVML_CLOCK_SM), int(get(h)), flush=True)
    time.sleep(0.004)
"""


class ClockSampler:
    """SM clock and clock-event (throttle) reasons sampled through NVML every ~5 ms by a SEPARATE process (a sampling thread in
    this process starves while the benchmark's Python thread runs); start() early, then window(t0, t1) keeps the samples whose
    wall-clock stamp lies inside the timed region.  Falls back to `nvidia-smi -lms` if NVML cannot be loaded."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    BITS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown", 0x4: "sw_power_cap",
            0x80: "hw_power_brake_slowdown"}

    def __init__(self, index):
        self.index = index
        self.lines = []
        self.proc = None
        self.mode = None

    def start(self):
        try:
            import pynvml  # noqa: F401  (the child needs it)
            try:
                import torch
                uuid = "GPU-" + str(torch.cuda.get_device_properties(self.index).uuid)
            except Exception:
                uuid = "-"
            self.proc = subprocess.Popen([sys.executable, "-c", _SAMPLER_SRC, uuid, str(self.index)], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.mode = "nvml"
        except Exception:
            try:
                self.proc = subprocess.Popen(
                    ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits", "-lms", "100"],
                    stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
                self.mode = "smi"
            except Exception:
                self.proc = None
        if self.proc:
            self.thread = threading.Thread(target=self._pump, daemon=True)
            self.thread.start()
            time.sleep(0.5)   # the child imports and initialises NVML before the timed region starts

    def _pump(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))

    def stop(self, t0=None, t1=None):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no clock sampler available"]}
        time.sleep(0.05)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        if self.mode == "nvml":
            mx, sm, mask = None, [], 0
            for _, ln in self.lines:
                f = ln.split()
                if len(f) == 2 and f[0] == "max":
                    mx = float(f[1])
                elif len(f) == 3:
                    t = float(f[0])
                    if (t0 is None or t >= t0) and (t1 is None or t <= t1):
                        sm.append(float(f[1]))
                        mask |= int(f[2])
            return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx, "samples": len(sm),
                    "reasons": sorted(nm for bit, nm in self.BITS.items() if mask & bit),
                    "source": "nvml in a sampler process, ~5 ms period, samples stamped inside the timed regions"}
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for t, ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 7 or (t0 is not None and t < t0) or (t1 is not None and t > t1 + 0.2):
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for nm, val in zip(names, f[3:7]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx,
                "samples": len(sm), "reasons": sorted(reasons), "source": "nvidia-smi -lms 100"}


def algorithmic_bytes(p, iters_hard):
    """Per-kernel algorithmic HBM bytes for a batch (uint8 entries)."""
    N, L = SHAPES[p]
    hard = int(iters_hard.size)
    ksum = int(iters_hard.sum())
    return {
        "delta": hard * L,                          # Delta written once
        "matrix": hard * (N * N + L),               # Delta gathered, M written once (first operator application fused: no extra bytes)
        # k_chain: the first application is fused into the builder and the LAST one of a surface only needs the cap row
        # (qfs_chain.cuh: cap_row_hit), so M is streamed max(0, k - 2) times per surface; plus a cap row per tested step and the vectors
        "matvec": int(np.maximum(iters_hard - 2, 0).sum()) * N * N + int(np.maximum(iters_hard - 1, 0).sum()) * N + ksum * N,
        # SURVEY.md 8d per-surface figure bytes(k) = N^2 + k N^2 + 2 L + (k+1) N, summed over the hard surfaces
        "total": hard * (N * N + 2 * L) + ksum * N * N + (ksum + hard) * N,
    }



def host_threads():
    """Host threads this process may use.  Not omp_get_max_threads(): torchrun exports OMP_NUM_THREADS=1 to its ranks, which
    would turn the CPU arm of an N > 1 run into a single-thread baseline."""
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except (AttributeError, OSError):
        return max(1, os.cpu_count() or 1)

def cpu_baseline(p, coeffs, budget_s):
    """C oracle (port of the reference CPU algorithm) on all host threads, on a bounded prefix."""
    import oracle
    threads = host_threads()
    pilot = min(len(coeffs), 8 * threads)
    t0 = time.perf_counter()
    oracle.heights_batch(coeffs[:pilot], p, 10, threads)
    dt = max(time.perf_counter() - t0, 1e-4)
    n = int(min(len(coeffs), max(pilot, pilot * budget_s / dt)))
    t0 = time.perf_counter()
    hs, _ = oracle.heights_batch(coeffs[:n], p, 10, threads)
    dt = time.perf_counter() - t0
    hard = int((hs != 1).sum())
    return {"value": n / dt, "unit": "surfaces/s", "cores": threads, "kind": "port",
            "hard_per_s": hard / dt,
            "sample": f"first {n} surfaces of the same seeded F_{p} batch ({hard} with height>=2), "
                      f"oracle/qfs_oracle.c (C port of qfsplit height_matrix), OpenMP over surfaces, {dt:.1f} s"}, hs


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    p = args.p
    coeffs = cached_block(p, min(args.batch, 20000), args.seed, 0)
    import oracle
    threads = host_threads()
    # size one step to ~ (120 s / (steps+warmup)) of CPU work
    pilot = 8 * threads
    t0 = time.perf_counter()
    oracle.heights_batch(coeffs[:pilot], p, 10, threads)
    per = (time.perf_counter() - t0) / pilot
    budget = 120.0 / max(1, args.steps + args.warmup)
    n = int(max(pilot, min(len(coeffs), budget / per)))
    for _ in range(args.warmup):
        oracle.heights_batch(coeffs[:n], p, 10, threads)
    t0 = time.perf_counter()
    hard = 0
    for _ in range(args.steps):
        hs, _ = oracle.heights_batch(coeffs[:n], p, 10, threads)
        hard = int((hs != 1).sum())
    dt = time.perf_counter() - t0
    val = n * args.steps / dt
    sample = (f"each step = first {n} surfaces of the seeded F_{p} batch ({hard} with height>=2) through "
              f"oracle/qfs_oracle.c (C port of the reference's qfsplit.height_matrix; the reference is pure "
              f"Python and is absent on the GPU box) on {threads} host threads")
    line = {
        "impl": "reference", "metric": "quartic K3 heights/sec", "value": val, "unit": "surfaces/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": {"workload": workload_name(p, args.batch), "p": p, "bound": 10},
        "cpu_baseline": {"value": val, "unit": "surfaces/s", "cores": threads, "kind": "port", "sample": sample,
                         "reference_python": reference_python_rate(p)},
        "e2e": {"value": val, "unit": "surfaces/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line))


def measure_gpu(p, batch, steps, warmup, seed, rank, world, device, dist):
    import torch
    from paper_2502_12428_b200.engine import get_engine
    eng = get_engine(p, device)
    host = cached_block(p, batch, seed, rank)
    pinned = torch.from_numpy(host).pin_memory()
    dev = pinned.to(f"cuda:{device}", non_blocking=False)
    hs = torch.empty(batch, dtype=torch.int8, device=dev.device)
    its = torch.empty(batch, dtype=torch.int8, device=dev.device)

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize(device)

    sampler = ClockSampler(device)
    sampler.start()
    for _ in range(warmup):
        eng.heights(dev, 10, out=(hs, its))
    stage = {"ms_power": 0.0, "ms_delta": 0.0, "ms_matrix": 0.0, "ms_matvec": 0.0, "ms_total": 0.0}
    launches = 0
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    wall0 = time.time()
    e0.record()
    for _ in range(steps):
        eng.heights(dev, 10, out=(hs, its))
        st = eng.stats()
        for k in stage:
            stage[k] += st[k]
        launches += st["kernel_launches"]
    e1.record()
    barrier()
    ms = e0.elapsed_time(e1)
    st = eng.stats()

    # end to end through the PUBLIC entry (height_batch: argument checks, host -> device copy of the batch, the pipeline, device ->
    # host copy of the results) with pinned host buffers; the clock sampler keeps running: same kernels, same load
    from paper_2502_12428_b200 import height_batch
    h_hs = torch.empty(batch, dtype=torch.int8).pin_memory().numpy()
    h_its = torch.empty(batch, dtype=torch.int8).pin_memory().numpy()
    h_in = pinned.numpy()
    e2e_steps = max(1, min(steps, 10))
    height_batch(p, h_in, 10, devices=[device], out=(h_hs, h_its))
    barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        height_batch(p, h_in, 10, devices=[device], out=(h_hs, h_its))
    torch.cuda.synchronize(device)
    e2e_s = time.perf_counter() - t0
    clocks = sampler.stop(wall0, time.time())

    heights = hs.cpu().numpy()
    iters = its.cpu().numpy()
    assert np.array_equal(heights, h_hs) and np.array_equal(iters, h_its)
    if dist is not None:
        t = torch.tensor([ms, e2e_s], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, e2e_s = float(t[0]), float(t[1])
    return {"ms": ms, "e2e_s": e2e_s, "e2e_steps": e2e_steps, "stage": stage, "launches": launches, "stats": st,
            "heights": heights, "iters": iters, "coeffs": host, "clocks": clocks}


def measure_single_surface(device, results):
    """BASELINE.json configs[0]: ONE quartic through the public call with host buffers (wall clock, median of 20), for the
    surface of the seeded batch with the most operator applications, next to the CPU oracle on one thread."""
    import oracle
    from paper_2502_12428_b200.engine import get_engine
    out = {}
    for p, res in results.items():
        i = int(np.argmax(res["iters"]))
        one = np.ascontiguousarray(res["coeffs"][i:i + 1])
        eng = get_engine(p, device)
        ts = []
        for k in range(23):
            t0 = time.perf_counter()
            h, it = eng.heights(one, 10)
            if k >= 3:
                ts.append(time.perf_counter() - t0)
        t0 = time.perf_counter()
        oh, oit = oracle.heights_batch(one, p, 10, 1)
        cpu_s = time.perf_counter() - t0
        out[f"F_{p}"] = {"ms_per_call": 1e3 * float(np.median(ts)), "height": int(h[0]), "iterations": int(it[0]),
                         "cpu_oracle_ms": 1e3 * cpu_s, "cpu_cores": 1,
                         "equals_oracle": bool(int(oh[0]) == int(h[0]) and int(oit[0]) == int(it[0])),
                         "surface": f"index {i} of the seeded batch", "stage_ms": {k: v for k, v in eng.stats().items() if k.startswith("ms_")}}
    return out


def measure_matrix_free(device, seed, checked):
    """surfaces/s of qfs_heights_free on resident inputs (CUDA events), F_5 ... F_13, 100000 seeded quartics each;
    for the primes in `checked` the heights and iteration counts are compared with the matrix path's."""
    import torch
    from paper_2502_12428_b200.engine import get_engine
    out = {"note": "polynomial iteration g <- -f^(p-2) u(Delta_1(f) g) without Delta and without the operator matrix "
                   "(csrc/qfs_free.cuh); same heights and iterations; not the path the roofline is quoted on"}
    for p in (5, 7, 11, 13):
        batch = 100000
        host = cached_block(p, batch, seed, 0)
        dev = torch.from_numpy(host).to(f"cuda:{device}")
        hs = torch.empty(batch, dtype=torch.int8, device=dev.device)
        its = torch.empty(batch, dtype=torch.int8, device=dev.device)
        eng = get_engine(p, device)
        for _ in range(3):
            eng.heights(dev, 10, out=(hs, its), matrix_free=True)
        torch.cuda.synchronize(device)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        steps = 5
        e0.record()
        for _ in range(steps):
            eng.heights(dev, 10, out=(hs, its), matrix_free=True)
        e1.record()
        torch.cuda.synchronize(device)
        ms = e0.elapsed_time(e1) / steps
        h = hs.cpu().numpy()
        entry = {"value": batch / (ms * 1e-3), "unit": "surfaces/s", "ms_per_step": ms, "batch": batch,
                 "hard_per_s": float((h != 1).sum()) / (ms * 1e-3)}
        if p in checked:
            entry["equals_matrix_path"] = bool(np.array_equal(h, checked[p]["heights"]) and
                                               np.array_equal(its.cpu().numpy(), checked[p]["iters"]))
        out[f"F_{p}"] = entry
    return out


def measure_lazy(device, seed, checked):
    """surfaces/s of the lazy operator-matrix mode (qfs_heights_lazy: the cap row of the first step decides before Delta and M
    are built) on resident inputs (CUDA events) and end to end through height_batch(method="lazy") with pinned host buffers;
    F_5, F_7 at 100000 seeded quartics, F_11 at 4000 and 20000, F_13 at 2000; heights and iterations compared with the eager path's."""
    import time
    import torch
    from paper_2502_12428_b200 import height_batch
    from paper_2502_12428_b200.engine import get_engine
    out = {"note": "the operator-matrix path with the loop's early exit (height.py:135-144) taken before the matrix is built: "
                   "(M g)[cap] is one row of M = N entries of Delta, evaluated from the factorised Witt carry (csrc/qfs_caprow.cuh); "
                   "Delta and M are built and streamed for the surfaces it leaves undecided only (built); same heights and "
                   "iterations; the headline and the roofline stay on the eager path, which builds M for every hard surface like the reference"}
    for p, batch in ((5, 100000), (7, 100000), (11, 4000), (11, 20000), (13, 2000)):
        host = cached_block(p, batch, seed, 0)
        dev = torch.from_numpy(host).to(f"cuda:{device}")
        hs = torch.empty(batch, dtype=torch.int8, device=dev.device)
        its = torch.empty(batch, dtype=torch.int8, device=dev.device)
        eng = get_engine(p, device)
        for _ in range(3):
            eng.heights(dev, 10, out=(hs, its), lazy=True)
        torch.cuda.synchronize(device)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        steps = 5
        e0.record()
        for _ in range(steps):
            eng.heights(dev, 10, out=(hs, its), lazy=True)
        e1.record()
        torch.cuda.synchronize(device)
        ms = e0.elapsed_time(e1) / steps
        st = eng.stats()
        h = hs.cpu().numpy()
        entry = {"value": batch / (ms * 1e-3), "unit": "surfaces/s", "ms_per_step": ms, "batch": batch,
                 "hard": int(st["hard"]), "built": int(st["built"]), "hard_per_s": float((h != 1).sum()) / (ms * 1e-3),
                 "stage_ms_per_step": {k: v for k, v in st.items() if k.startswith("ms_")}}
        # end to end: pinned host buffers in and out through the public entry
        pin_c = torch.from_numpy(host).pin_memory()
        pin_h = torch.empty(batch, dtype=torch.int8).pin_memory()
        pin_i = torch.empty(batch, dtype=torch.int8).pin_memory()
        for _ in range(2):
            height_batch(p, pin_c.numpy(), 10, devices=[device], method="lazy", out=(pin_h.numpy(), pin_i.numpy()))
        t0 = time.perf_counter()
        for _ in range(steps):
            height_batch(p, pin_c.numpy(), 10, devices=[device], method="lazy", out=(pin_h.numpy(), pin_i.numpy()))
        entry["e2e"] = {"value": batch * steps / (time.perf_counter() - t0), "unit": "surfaces/s", "h2d_bytes_per_step": 35 * batch,
                        "d2h_bytes_per_step": 2 * batch, "through": "height_batch(method='lazy'), pinned host buffers, host clock around the calls"}
        eager = None
        if p in checked and checked[p]["heights"].shape[0] == batch:
            eager = (checked[p]["heights"], checked[p]["iters"])
        else:
            eh, ei = eng.heights(dev, 10)
            eager = (eh.cpu().numpy(), ei.cpu().numpy())
        entry["equals_eager_matrix_path"] = bool(np.array_equal(h, eager[0]) and np.array_equal(its.cpu().numpy(), eager[1]) and
                                                 np.array_equal(pin_h.numpy(), eager[0]) and np.array_equal(pin_i.numpy(), eager[1]))
        out[f"F_{p}" + ("" if (p, batch) != (11, 20000) else "_20000")] = entry
    return out


def gpu_line(args, p, res, world, with_cpu):
    batch, steps = args.batch, res["steps"]
    peak, peak_src = measured_peaks()
    heights, iters = res["heights"], res["iters"]
    hard_mask = heights != 1
    hard = int(hard_mask.sum())
    ab = algorithmic_bytes(p, iters[hard_mask].astype(np.int64))
    ms_step = res["ms"] / steps
    value = world * batch * steps / (res["ms"] * 1e-3)
    stage = {k: v / steps for k, v in res["stage"].items()}
    kernels = {"delta": ("k_delta_mma", stage["ms_delta"], ab["delta"]),
               "matrix": ("k_matrix_staged", stage["ms_matrix"], ab["matrix"]),
               "matvec": ("k_chain" if p <= 7 else "k_chain_grid", stage["ms_matvec"], ab["matvec"])}
    top = max(kernels, key=lambda k: kernels[k][1])
    name, kms, kbytes = kernels[top]
    ach = kbytes / (kms * 1e-3) / 1e9 if kms > 0 else 0.0
    N, L = SHAPES[p]
    line = {
        "metric": "quartic K3 heights/sec", "value": value, "unit": "surfaces/s", "n_gpus": world,
        "steps": steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": (value * hard / batch) / PAPER_RATE[p] if p in PAPER_RATE else None,
        "dtype": "u8", "data": "synthetic",
        "config": {
            "workload": workload_name(p, batch),
            "p": p, "batch_per_gpu": batch, "seed": args.seed, "parallelism": f"{world} independent shards, no collective",
            "l2": f"working set per step {ab['total'] / 1e9:.1f} GB >> 126 MB L2 (no flush needed)",
            "vs_baseline_note": "hard (height>=2) surfaces/s over the paper's " + PAPER_NOTE.get(p, "(no published figure)") + " (BASELINE.md s1)",
        },
        "hard_fraction": hard / batch,
        "hard_per_s": value * hard / batch,
        "height_histogram": {str(k): int(v) for k, v in enumerate(np.bincount(heights.astype(np.int64), minlength=2)) if v},
        "stage_ms_per_step": stage,
        "roofline": {"bound": "hbm", "kernel": name, "achieved": ach, "peak": peak, "unit": "GB/s",
                     "frac": ach / peak, "traffic": measured_traffic(p, name, hard, max(1, res["stats"]["chunks"])),
                     "algorithmic_bytes_per_launch": kbytes / max(1, res["stats"]["chunks"]),
                     "launches_per_step": res["stats"]["chunks"], "ms_per_step": kms, "peak_source": peak_src,
                     "all_kernels": {k: {"ms": v[1], "GBps": (v[2] / (v[1] * 1e-3) / 1e9 if v[1] > 0 else 0.0)} for k, v in kernels.items()}},
        "roofline_pipeline": {"algorithmic_bytes_per_step": ab["total"], "achieved": ab["total"] / (ms_step * 1e-3) / 1e9,
                              "peak": peak, "unit": "GB/s", "frac": ab["total"] / (ms_step * 1e-3) / 1e9 / peak,
                              "note": "SURVEY 8d bytes of the reference's algorithm (M read once per operator application); the engine "
                                      "moves fewer -- the first application is fused into the builder and the last one of a surface reads "
                                      "one row -- so this figure may exceed 1; the per-kernel roofline above is the one to read"},
        "e2e": {"value": world * batch * res["e2e_steps"] / res["e2e_s"], "unit": "surfaces/s",
                "h2d_bytes_per_step": batch * 35, "d2h_bytes_per_step": 2 * batch,
                "through": "paper_2502_12428_b200.height_batch (the public entry), pinned host buffers"},
        "gpu_launches": int(res["launches"]),
        "clocks": res["clocks"],
    }
    if with_cpu:
        cb, ohs = cpu_baseline(p, res["coeffs"], args.cpu_seconds)
        n = len(ohs)
        cb["parity_on_sample"] = bool(np.array_equal(ohs, heights[:n]))
        cb["reference_python"] = reference_python_rate(p)
        line["cpu_baseline"] = cb
    return line


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200")
    ap.add_argument("--p", type=int, default=5)
    ap.add_argument("--batch", type=int, default=100000)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-also", action="store_true", help="skip the secondary F_7 measurement")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 0)

    if args.impl == "reference":
        run_reference_arm(args)
        return

    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if os.environ.get("QFS_BENCH_SHARE_GPU"):
        local = 0   # test hook: every rank on cuda:0, to exercise the N > 1 path on a one-GPU box (not a measurement)
    dist = None
    if world > 1:
        import torch.distributed as dist_mod
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        torch.cuda.set_device(local)
        dist_mod.init_process_group("gloo")   # a barrier and one 2-double max: the path itself has no collective (no NCCL)
        dist = dist_mod
    elif args.gpus > 1 and "RANK" not in os.environ:
        # convenience: relaunch under torchrun
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", "29531"] + sys.argv
        sys.exit(subprocess.call(cmd))
    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device (there is no CPU fallback); use --impl reference for the CPU arm")
    torch.cuda.set_device(local)

    res = measure_gpu(args.p, args.batch, args.steps, max(args.warmup, 3), args.seed, rank, world, local, dist)
    res["steps"] = args.steps
    line = None
    if rank == 0:
        line = gpu_line(args, args.p, res, world, with_cpu=True)
    if not args.no_also and args.p == 5:
        keep = ("value", "unit", "ms_per_step", "steps", "hard_per_s", "vs_baseline", "stage_ms_per_step", "roofline",
                "roofline_pipeline", "e2e", "cpu_baseline", "height_histogram", "config", "clocks")
        k7 = max(2, args.steps // 3)
        # every configuration gets the device's memory to itself, as a user running it alone would: the engines of the
        # previous configuration (and their HBM workspaces, which size the next engine's chunks) are closed first
        from paper_2502_12428_b200.engine import close_all
        close_all()
        res7 = measure_gpu(7, args.batch, k7, 3, args.seed, rank, world, local, dist)
        res7["steps"] = k7
        if rank == 0:
            l7 = gpu_line(args, 7, res7, world, with_cpu=(world == 1))
            line["also"] = {"F_7": {k: l7[k] for k in keep if k in l7}}
        # BASELINE.json configs[4]: F_11 (12341 x 12341 operator, 152 MB per matrix): a batch sized so that its
        # ~9% hard surfaces fill one HBM-budgeted chunk; no CPU arm (the oracle needs minutes per F_11 surface)
        b11 = min(args.batch, 4000)
        saved = args.batch
        args.batch = b11
        close_all()
        res11 = measure_gpu(11, b11, 5, 3, args.seed, rank, world, local, dist)
        res11["steps"] = 5
        if rank == 0:
            l11 = gpu_line(args, 11, res11, world, with_cpu=False)
            line["also"]["F_11"] = {k: l11[k] for k in keep if k in l11}
        args.batch = saved
        # The matrix-free iteration (qfs_heights_free): same heights and iteration counts, no Delta, no M.  NOT the contract
        # path (the north star requires the operator matrix in HBM and the streamed matvec chain): reported beside it.
        if rank == 0 and world == 1:
            line["also"]["matrix_free"] = measure_matrix_free(local, args.seed, {5: res, 7: res7})
            line["also"]["single_surface"] = measure_single_surface(local, {5: res, 7: res7})
            line["also"]["lazy_matrix"] = measure_lazy(local, args.seed, {5: res, 7: res7})
    if rank == 0:
        print(json.dumps(line))
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
