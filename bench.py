"""Benchmark: (kernel x freq-pair) evals/s of the fused DSO hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3|c2|c4] [--impl ours|reference]

Default workload (config c3, BASELINE.json configs[2]): per GPU 16,777,216
synthetic kernels (gen_kernel stream, generated on the device) x 128 core x 4
memory frequencies, eta = 0.8.  One step = the whole hot path over the batch:
raw PTX counts + DCGM -> feature normalisation/fusion -> MLP (134-100-50-25-7)
-> P(f), T(f) over the 512-pair grid -> eta objective -> argmin, in ONE fused
kernel launch.  Weak scaling: every rank runs its own 16M-kernel shard of the
global stream (no data-path collective; barrier + max-over-ranks timing only).

Timed with CUDA events on the launching stream; inputs (8.6 GB/GPU) exceed the
126 MB L2, so no flush is needed.  `e2e` re-measures the same metric through
the C-ABI with pinned HOST buffers (H2D + compute + D2H inside the call).
`--impl reference` times the CPU reference path on the host's cores instead.
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

METRIC = "(kernel×freq-pair) evals/sec, 1/2/4/8 B200, % roofline vs host-CPU ref"
UNIT = "(kernel, freq-pair) evals/s"
ROOT_SEED = 0xD50B203
DSO_COUNT_ROWS = 126
MLP_FLOPS = 2 * (134 * 100 + 100 * 50 + 50 * 25 + 25 * 7)  # 39,650 per kernel
PAIR_FLOPS = 14


def mlp_flops_sparse(l1_rows):
    """MLP flops per kernel when layer 1 sees l1_rows non-zero inputs."""
    return 2 * (l1_rows * 100 + 100 * 50 + 50 * 25 + 25 * 7)
CONFIGS = {
    "c2": dict(n=1 << 20, nc=64, nm=1, eta=0.8,
               desc="C2: 1M kernels x 64 core x 1 mem freqs, eta 0.8"),
    "c3": dict(n=1 << 24, nc=128, nm=4, eta=0.8,
               desc="C3: 16M kernels x 128 core x 4 mem freqs per GPU, eta 0.8"),
    "c4": dict(n=1 << 22, nc=128, nm=4, eta=None,
               desc="C4: 101 etas (0.00..1.00) x 4M kernels x 128 core x 4 mem"),
    "c5": dict(n=10_000_000, nc=128, nm=4, eta=None, batch=65536,
               desc="C5: predictor training, 10M synthetic samples per GPU, "
                    "65,536-sample batch per GPU, NCCL grad allreduce"),
}
TRAIN_FLOPS = 92_150  # per sample-step, SURVEY.md §8(d)


def env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--kernels", type=int, default=0, help="override kernels per GPU")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-stages", action="store_true")
    ap.add_argument("--no-extra", action="store_true",
                    help="skip the other configs (C2, C4, C5) measured after the headline")
    ap.add_argument("--cpu-sample", type=int, default=0)
    ap.add_argument("--engine", default="auto", choices=["auto", "ffma", "tc"],
                    help="predictor engine: the library's auto choice (tcgen05 for CSR), "
                         "the FMA-pipe kernel, or the tcgen05 3xTF32 kernel")
    ap.add_argument("--input", default="csr", choices=["csr", "dense"],
                    help="PTX counts as sparse per-kernel lists (the reference's map shape) "
                         "or dense [126][n] rows")
    return ap.parse_args()


# ---------------------------------------------------------------------------------------
class ClockSampler:
    """SM clocks + throttle reasons sampled (NVML, every 10 ms; nvidia-smi as a
    fallback) during the timed region."""

    def __init__(self, gpus):
        self.gpus = gpus
        self.rows = []
        self.stop = threading.Event()
        self.t = None

    def _nvml(self):
        import pynvml as N
        N.nvmlInit()
        hs = [(g, N.nvmlDeviceGetHandleByIndex(g)) for g in self.gpus]
        bits = {"hw_slowdown": N.nvmlClocksThrottleReasonHwSlowdown,
                "hw_thermal_slowdown": N.nvmlClocksThrottleReasonHwThermalSlowdown,
                "sw_thermal_slowdown": N.nvmlClocksThrottleReasonSwThermalSlowdown,
                "sw_power_cap": N.nvmlClocksThrottleReasonSwPowerCap}
        while not self.stop.is_set():
            for g, h in hs:
                try:
                    sm = N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)
                    mx = N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM)
                    pw = N.nvmlDeviceGetPowerUsage(h) / 1000.0
                    rs = N.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                    self.rows.append((g, sm, mx, pw, [k for k, v in bits.items() if rs & v]))
                except N.NVMLError:
                    pass
            self.stop.wait(0.01)
        N.nvmlShutdown()

    def __enter__(self):
        try:
            import pynvml  # noqa: F401
            self.t = threading.Thread(target=self._nvml, daemon=True)
            self.t.start()
        except ImportError:
            self.t = None
        return self

    def __exit__(self, *exc):
        self.stop.set()
        if self.t:
            self.t.join(timeout=2)

    def summary(self):
        rows = self.rows
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(r[1] for r in rows),
                "sm_max_mhz": max(r[2] for r in rows),
                "reasons": sorted({x for r in rows for x in r[4]}),
                "samples": len(rows), "power_w_max": max(r[3] for r in rows),
                "sampler": "NVML every 10 ms during the timed region"}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except (OSError, ValueError):
        return {}


def ncu_traffic(config, n):
    """DRAM bytes (read + write) per launch of the dominant kernel, from the committed
    ncu --set full capture (profiles/ncu_summary.json), scaled to this launch's n."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            e = json.load(f).get(config, {})
        if e.get("dram_bytes_per_kernel") is None:
            return None
        return e["dram_bytes_per_kernel"] * n
    except (OSError, ValueError):
        return None


# ---------------------------------------------------------------------------------------
def ref_domain(nc, nm):
    """The benchmark grid without the product package: fc = 705 +
    675 i/(nc-1), fm = 438 + 439 j/(nm-1) or {877}; default_device (sim_harness.cpp:103-106)
    as [kappa_vf, pmax, vmin, vmax, mhz_per_unit]."""
    core = 705.0 + (1380.0 - 705.0) * np.arange(nc) / max(nc - 1, 1)
    mem = np.array([877.0]) if nm == 1 else 438.0 + 439.0 * np.arange(nm) / (nm - 1)
    return core, mem, np.array([0.5, 300.0, 0.55, 2.10, 1000.0])


def cpu_pipeline_rate(port, ref, n, cfg, model, threads):
    """Host-CPU reference path on n kernels: features + MLP (C restatement; the
    reference needs Eigen, absent) and brute_force_config (the reference's own
    optimizer.cpp, oracle/_ref).  Returns (pairs/s, seconds, detail)."""
    core, mem, dev = ref_domain(cfg["nc"], cfg["nm"])
    g = port.gen_stream(ROOT_SEED, n, want=("counts", "dcgm"), threads=threads)
    t0 = time.perf_counter()
    fused = port.fuse(g["counts"], g["dcgm"])
    params, _ = port.predict_params(model, fused, threads=threads)
    t1 = time.perf_counter()
    eta = cfg["eta"] if cfg["eta"] is not None else 0.8
    if ref is not None:
        ref.brute_force_config(params, core, mem, dev, eta, dev[1], threads=threads)
        sweep_kind = "reference optimizer.cpp (oracle/_ref)"
    else:
        port.brute_force(params, core, mem, dev, eta, dev[1], threads=threads)
        sweep_kind = "C restatement (oracle/liboracle.so)"
    t2 = time.perf_counter()
    pairs = n * len(core) * len(mem)
    return pairs / (t2 - t0), t2 - t0, {"features_mlp_s": t1 - t0, "sweep_s": t2 - t1,
                                         "sweep_impl": sweep_kind}


class OracleModel:
    """A model object in the layout the oracle reads (layer_sizes, weights, biases,
    target_mean, target_std) — the reference arm never touches the product library."""

    def __init__(self, layer_sizes, weights, biases, target_mean, target_std):
        self.layer_sizes, self.weights, self.biases = layer_sizes, weights, biases
        self.target_mean, self.target_std = target_mean, target_std


def bench_model(port):
    """Model for the CPU legs: init_mlp(default_layer_sizes, 424242) by the oracle's
    restatement of mlp.cpp:184-207 (identical draws to the device model), with the
    population mean / std of 65,536 synthetic truth parameters as target stats."""
    sizes = [134, 100, 50, 25, 7]
    ws, bs = port.init_mlp(sizes, 424242)
    p = port.gen_stream(0xC0FFEE, 65536, want=("params",))["params"]
    return OracleModel(sizes, ws, bs, p.mean(0), p.std(0))


def run_reference(args, rank, world):
    if rank != 0:
        return
    import oracle
    port = oracle.port()
    try:
        ref = oracle.ref()
    except (FileNotFoundError, OSError):
        ref = None
    cfg = CONFIGS[args.config]
    threads = oracle.oracle.default_threads()
    n = args.cpu_sample or 65536
    model = bench_model(port)
    for _ in range(max(args.warmup, 0)):
        cpu_pipeline_rate(port, ref, min(n, 4096), cfg, model, threads)
    rates, secs = [], []
    for _ in range(args.steps):
        r, s, det = cpu_pipeline_rate(port, ref, n, cfg, model, threads)
        rates.append(r)
        secs.append(s)
    total_pairs = n * cfg["nc"] * cfg["nm"] * args.steps
    value = total_pairs / sum(secs)
    sample = (f"{n} kernels/step of the {args.config} workload ({cfg['desc']}); features+MLP: "
              f"C restatement (reference needs Eigen, absent); sweep: {det['sweep_impl']}")
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * sum(secs) / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (gen_kernel stream)", "impl": "reference",
        "config": {"workload": cfg["desc"], "kernels_per_step": n},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads,
                         "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------------------
TC_L1_FLOPS = 3 * 2 * 128 * 112 * 8   # one tcgen05 layer-1 k-step: 3 kind::tf32 MMAs M128 N112 K8
TC_L2_FLOPS = 3 * 2 * 128 * 64 * 8    # one layer-2 k-step: 3 MMAs M128 N64 K8


def cuda_time(stream, fn, reps):
    """Mean ms per call of fn over reps calls, CUDA events on the launching stream."""
    import torch
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record(stream)
    for _ in range(reps):
        fn()
    b.record(stream)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


class Timed:
    """W warm-up steps, then K steps between barrier + synchronize, CUDA events on
    the launching stream, max over ranks (the contract's timing rule)."""

    def __init__(self, world, dev, stream):
        self.world, self.dev, self.stream = world, dev, stream

    def barrier(self):
        if self.world > 1:
            import torch.distributed as dist
            dist.barrier()

    def max_over_ranks(self, v):
        import torch
        import torch.distributed as dist
        t = torch.tensor([v], dtype=torch.float64, device=self.dev)
        if self.world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def run(self, step, steps, warmup, clocks=None):
        import torch
        for i in range(warmup):
            step(i)
        torch.cuda.synchronize()
        self.barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(self.stream)
        for i in range(steps):
            step(warmup + i)
        e1.record(self.stream)
        torch.cuda.synchronize()
        self.barrier()
        ms = e0.elapsed_time(e1) / steps
        return ms, self.max_over_ranks(ms)


def fp32_peak(ctx):
    """Builder-measured FP32 peaks (dso_probe_fp32_peak: FFMA2 / FFMA loops on
    148 x 4 CTAs). MEASURED_PEAKS.json has no FP32 figure."""
    import ctypes as C
    from paper_2407_13096_b200 import _lib
    out = {}
    for mode, name in ((1, "ffma2"), (0, "ffma")):
        v = C.c_double()
        ctx._raise(_lib.lib().dso_probe_fp32_peak(ctx._h, mode, C.byref(v)))
        out[name] = v.value
    return out


PEAK_NOTE = ("builder-measured in this run: dso_probe_fp32_peak (FFMA2 loop on 148x4 CTAs); "
             "MEASURED_PEAKS.json has no FP32 figure")


def measure_pipeline(ctx, name, args, rank, world, tm, peak, steps, warmup, csr=True,
                     with_e2e=False, clocks=None):
    """C2 / C3: the fused pipeline (features -> MLP -> sweep -> argmin) over this rank's
    shard of the synthetic stream.  Returns (line fields, inputs)."""
    import torch
    from paper_2407_13096_b200 import linear_domain
    cfg = CONFIGS[name]
    n = args.kernels if (args.kernels and name == args.config) else cfg["n"]
    dom = linear_domain(cfg["nc"], cfg["nm"])
    ctx.set_domain(dom)
    if csr:
        gen = ctx.gen_synthetic_csr(n, root=ROOT_SEED, first=rank * n)
        dcgm = gen["dcgm"]
        nnz = float((gen["row_ptr"][n] - gen["row_ptr"][0]).item()) / n
    else:
        gen = ctx.gen_synthetic(n, root=ROOT_SEED, first=rank * n, params=False)
        dcgm = gen["dcgm"]
        # the algorithmic layer-1 work counts the listed (non-zero) categories, whatever
        # the input format
        nnz = float((gen["counts"] != 0).sum().item()) / n
    out = ctx.alloc_pipeline_out(n)
    if csr:
        step = lambda i: ctx.pipeline_csr(gen["row_ptr"], gen["entries"], dcgm, cfg["eta"], out=out)  # noqa: E731
    else:
        step = lambda i: ctx.pipeline(gen["counts"], dcgm, cfg["eta"], out=out)  # noqa: E731
    launches0 = ctx.launch_count
    ctx.counters(reset=True)
    for i in range(warmup):
        step(i)
    ctx.counters(reset=True)
    launches0 = ctx.launch_count
    if clocks is not None:
        with clocks:
            ms, ms_max = tm.run(step, steps, 0)
    else:
        ms, ms_max = tm.run(step, steps, 0)
    ctr = ctx.counters(reset=True)
    launches = ctx.launch_count - launches0
    pairs = dom.pairs
    units = n * pairs
    value = units * world / (ms_max * 1e-3)
    # FP32-equivalent algorithmic work, layer 1 on the rows a
    # kernel lists (8 DCGM + its non-zero count slots; all-zero rows are exact zeros)
    fpk = mlp_flops_sparse(8 + nnz) + PAIR_FLOPS * pairs
    fpk_dense = MLP_FLOPS + PAIR_FLOPS * pairs
    achieved = n * fpk / (ms * 1e-3) / 1e12
    peaks = measured_peaks()
    engine = "tc" if ctr["tc_tiles"] > 0 else "ffma"
    roofline = {
        "bound": "fp32", "achieved": achieved, "peak": peak["ffma2"], "unit": "TFLOP/s",
        "frac": achieved / peak["ffma2"],
        "traffic": ncu_traffic(name, n) if csr else None,
        "traffic_unit": "bytes per launch (ncu dram__bytes_read+write, profiles/ncu_summary.json)",
        "algorithmic_bytes_per_launch": n * ((8 + 4 * nnz + 32) if csr else (126 * 4 + 32)) + n * 16,
        "kernel": ("tc_kernel<MODE_CSR> (fused pipeline; layers 1-2 on tcgen05 kind::tf32)"
                   if engine == "tc" else "ws_kernel (fused pipeline, FFMA2)"),
        "flops_per_kernel": fpk,
        "flops_note": ("FP32-equivalent algorithmic flops per kernel: MLP with layer 1 on the 8 + "
                       f"{nnz:g} listed input rows (2*100*(8+nnz) + 2*(5000+1250+175)) + "
                       f"{PAIR_FLOPS} per (kernel, pair) x {pairs} pairs; the dense-input count "
                       "(SURVEY.md §8(d)) is flops_per_kernel_dense"),
        "flops_per_kernel_dense": fpk_dense,
        "peak_source": PEAK_NOTE, "peak_ffma_scalar": peak["ffma"],
        "nominal_peak": 148 * 128 * 2 * peaks.get("sm_max_mhz", 1965.0) * 1e6 / 1e12,
        "binding_unit": "CUDA-core issue (FP32/ALU pipes): producers' CSR feature stage and the "
                        "epilogues' layers 3-4 + grid sweep; the tensor pipe is not the limiter "
                        "(tensor_view)",
    }
    if engine == "tc":
        issued = ctr["tc_l1_ksteps"] * TC_L1_FLOPS + ctr["tc_l2_ksteps"] * TC_L2_FLOPS
        tflops = issued / steps / (ms * 1e-3) / 1e12
        tpk = peaks.get("bf16_tflops", 2250.0) / 2
        roofline["tensor_view"] = {
            "achieved": tflops, "peak": tpk, "frac": tflops / tpk, "unit": "TFLOP/s",
            "issued_flops_per_step": issued / steps,
            "l1_ksteps_per_tile": ctr["tc_l1_ksteps"] / max(ctr["tc_tiles"], 1),
            "l2_ksteps_per_tile": ctr["tc_l2_ksteps"] / max(ctr["tc_tiles"], 1),
            "source": "device counters (dso_get_counters) over the timed steps: k-steps the MMA "
                      "thread issued x 3 kind::tf32 MMAs (M128 x N112 x K8 layer 1, "
                      "M128 x N64 x K8 layer 2; padded shapes)",
            "peak_source": "MEASURED_PEAKS.json bf16_tflops / 2 (dense TF32 = half the bf16 rate)",
        }
    res = {"value": value, "unit": UNIT, "ms_per_step": ms_max, "steps": steps,
           "kernels_per_gpu": n, "grid": f"{cfg['nc']}x{cfg['nm']}", "engine": engine,
           "roofline": roofline, "gpu_launches": launches,
           "input": ("sparse per-kernel PTX count lists (%g non-zeros/kernel) + DCGM" % nnz
                     if csr else "dense [126][n] PTX counts (%g non-zeros/kernel) + DCGM; auto "
                     "engine: compacted to CSR on the device, tensor-core CSR pipeline" % nnz)}
    if with_e2e:
        res["e2e"] = measure_e2e(ctx, gen, dcgm, cfg, n, csr, steps, tm, world, units)
    return res, gen


def measure_e2e(ctx, gen, dcgm, cfg, n, csr, steps, tm, world, units):
    """The same metric through the C-ABI with pinned HOST buffers (H2D + kernel + D2H
    inside each timed call)."""
    hd = dcgm.cpu().pin_memory()
    if csr:
        hrp = gen["row_ptr"].cpu().pin_memory()
        hent = gen["entries"].cpu().pin_memory()
        h2d = (n + 1) * 8 + hent.numel() * 4 + n * 8 * 4
        run = lambda o: ctx.pipeline_csr(hrp, hent, hd, cfg["eta"], out=o)  # noqa: E731
    else:
        hc = gen["counts"].cpu().pin_memory()
        h2d = n * (126 * 4 + 8 * 4)
        run = lambda o: ctx.pipeline(hc, hd, cfg["eta"], out=o)  # noqa: E731
    hout = ctx.alloc_pipeline_out(n, host=True, like=hd)
    run(hout)  # warm-up (staging buffers)
    k = max(1, min(steps, 5))
    tm.barrier()
    t0 = time.perf_counter()
    for _ in range(k):
        run(hout)
    el = tm.max_over_ranks((time.perf_counter() - t0) / k)
    probe = pcie_probe(hent if csr else hc)
    return {"value": units * world / el, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(n * 16), "ms_per_step": el * 1e3, "steps": k,
            "h2d_gbs": h2d / el / 1e9, "link": probe,
            "link_frac": (h2d / el / 1e9) / probe["h2d_gbs"] if probe.get("h2d_gbs") else None,
            "timing": "host wall clock around synchronous C-ABI calls (dso_pipeline%s with "
                      "DSO_HOST, pinned buffers), max over ranks" % ("_csr" if csr else "")}


def pcie_probe(host_buf):
    """The box's host->device copy bandwidth: plain cudaMemcpy of the same pinned
    buffer (the PCIe placement varies between boxes; e2e is judged against it)."""
    import torch
    try:
        src = host_buf.view(-1)[: min(host_buf.numel(), 1 << 28)]
        dst = torch.empty(src.shape, dtype=src.dtype, device="cuda")
        dst.copy_(src, non_blocking=True)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(3):
            dst.copy_(src, non_blocking=True)
        b.record()
        torch.cuda.synchronize()
        nbytes = src.numel() * src.element_size()
        gbs = 3 * nbytes / (a.elapsed_time(b) * 1e-3) / 1e9
        del dst
        return {"h2d_gbs": gbs, "bytes": nbytes, "method": "3 x torch copy_ of the pinned entry buffer, CUDA events"}
    except Exception as e:  # noqa: BLE001
        return {"error": str(e)[:120]}


def measure_eta(ctx, args, rank, world, tm, peak, steps, warmup):
    """C4: brute_force_config at 101 etas (dso_eta_sweep) over 4M kernels' params."""
    import ctypes as C

    import torch
    from paper_2407_13096_b200 import linear_domain
    from paper_2407_13096_b200.api import _ptr
    cfg = CONFIGS["c4"]
    n = args.kernels if (args.kernels and args.config == "c4") else cfg["n"]
    dom = linear_domain(cfg["nc"], cfg["nm"])
    ctx.set_domain(dom)
    params = ctx.gen_synthetic(n, root=ROOT_SEED, first=rank * n, counts=False, dcgm=False)["params"]
    dev = params.device
    idx_o = torch.empty((101, n), dtype=torch.int32, device=dev)
    cost_o = torch.empty((101, n), dtype=torch.float32, device=dev)
    etas = np.ascontiguousarray(np.arange(101) / 100.0)
    dp = C.POINTER(C.c_double)

    def step(i):
        ctx._raise(ctx._lib.dso_eta_sweep(ctx._h, _ptr(params), n, n, etas.ctypes.data_as(dp),
                                          101, dom.dev.pmax_w, _ptr(idx_o), _ptr(cost_o), n))
    for i in range(warmup):
        step(i)
    l0 = ctx.launch_count
    ms, ms_max = tm.run(step, steps, 0)
    units = n * dom.pairs
    fl = units * (9 + 3 * 101)
    achieved = fl / (ms * 1e-3) / 1e12
    return {"value": units * world / (ms_max * 1e-3), "unit": UNIT, "ms_per_step": ms_max,
            "steps": steps, "triples_per_s": units * 101 * world / (ms_max * 1e-3),
            "kernels_per_gpu": n, "grid": f"{cfg['nc']}x{cfg['nm']}", "gpu_launches": ctx.launch_count - l0,
            "roofline": {"bound": "fp32", "achieved": achieved, "peak": peak["ffma2"],
                         "frac": achieved / peak["ffma2"], "unit": "TFLOP/s",
                         "kernel": "eta_sweep_pruned_kernel",
                         "flops_per_pair": 9 + 3 * 101,
                         "flops_note": "P (3 FMA), T (mul, max, add), E (mul) once per (kernel, pair) "
                                       "= 9, plus C = (eta*P + K)*T = 3 per (kernel, pair, eta), over "
                                       "all nc*nm pairs (the brute-force work SURVEY.md 8(d) counts)",
                         "executed_view": {
                             "pairs_per_kernel": cfg["nc"] + cfg["nm"],
                             "achieved": n * (cfg["nc"] + cfg["nm"]) * (9 + 3 * 101) / (ms * 1e-3) / 1e12,
                             "frac": n * (cfg["nc"] + cfg["nm"]) * (9 + 3 * 101) / (ms * 1e-3) / 1e12
                                     / peak["ffma2"],
                             "note": "the pruned sweep evaluates only the nc + nm pairs no other pair "
                                     "can beat (sweep.cu; exact); its per-eta group minima, "
                                     "bookkeeping and winning-group replay run on the ALU pipe, "
                                     "the busiest unit (ncu)"},
                         "peak_source": PEAK_NOTE,
                         "traffic": ncu_traffic("c4", n),
                         "algorithmic_bytes_per_launch": n * (28 + 101 * 8)}}


def measure_train(ctx, args, rank, world, tm, peak, steps, warmup, model):
    """C5: synchronous data-parallel SGD steps (device gradient -> NCCL allreduce of
    the 20,007-float gradient -> identical device update) over a device-resident
    shard of synthetic samples per GPU."""
    import torch
    from paper_2407_13096_b200 import linear_domain
    cfg = CONFIGS["c5"]
    n = args.kernels if (args.kernels and args.config == "c5") else cfg["n"]
    ctx.set_domain(linear_domain(cfg["nc"], cfg["nm"]))
    ctx.set_model(model)
    dev = torch.device("cuda", ctx.device)
    B = cfg["batch"]
    gen = ctx.gen_synthetic(n, root=0xACCE5505, first=rank * n)
    x = ctx.featurize(gen["counts"], gen["dcgm"])
    del gen["counts"]
    p = gen["params"].double()
    mean = torch.tensor(model.target_mean, dtype=torch.float64, device=dev)
    std = torch.tensor(model.target_std, dtype=torch.float64, device=dev)
    y = ((p - mean[:, None]) / std[:, None]).float().contiguous()
    del p, gen
    from paper_2407_13096_b200.api import NcclComm
    comm = NcclComm(ctx.device) if world > 1 else None  # the library's own NCCL communicator
    nb = n // B
    grad = torch.empty((ctx.n_model_params,), dtype=torch.float32, device=dev)

    def step(i):
        # dso_train_step: gradient -> ncclAllReduce (in the library) -> update
        ctx.train_step(x, y, 0.1, B * world, n=B, start=(i % nb) * B, comm=comm, want_loss=False)

    for i in range(warmup):
        step(i)
    l0 = ctx.launch_count
    ms, ms_max = tm.run(step, steps, 0)
    launches = ctx.launch_count - l0
    grad_ms = cuda_time(tm.stream, lambda: ctx.train_grad_slice(x, y, 0, B, grad=grad), 5)
    achieved = B * TRAIN_FLOPS / (grad_ms * 1e-3) / 1e12
    step_tflops = B * TRAIN_FLOPS / (ms * 1e-3) / 1e12
    ctx.set_model(model)  # training moved the weights
    del x, y
    if comm is not None:
        comm.close()
    return {"metric": "predictor training sample-steps/s (C5)", "value": B * world / (ms_max * 1e-3),
            "unit": "samples/s", "ms_per_step": ms_max, "steps": steps,
            "samples_per_gpu": n, "batch_per_gpu": B, "global_batch": B * world,
            "parallelism": f"dp{world} (%s allreduce)" % ("NCCL" if world > 1 else "no"),
            "gpu_launches": launches,
            "roofline": {"bound": "fp32", "achieved": step_tflops, "peak": peak["ffma2"],
                         "frac": step_tflops / peak["ffma2"], "unit": "TFLOP/s",
                         "note": "whole step (gradient kernels, allreduce when N > 1, update)",
                         "grad_call_view": {"achieved": achieved, "frac": achieved / peak["ffma2"],
                                            "note": "dso_train_grad alone, back-to-back calls "
                                                    "(includes per-call host overhead)"},
                         "traffic": ncu_traffic("c5", B),
                         "traffic_unit": "bytes per dso_train_grad (ncu, profiles/ncu_summary.json)",
                         "kernel": "dso_train_grad kernels (step: dso_train_step)", "flops_per_sample": TRAIN_FLOPS,
                         "grad_kernel_ms": grad_ms, "peak_source": PEAK_NOTE}}


def run_ours(args, rank, world, local_rank):
    import torch

    from paper_2407_13096_b200.api import Context

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    ctx = Context(local_rank)
    ctx.set_option("mlp_engine", {"ffma": 0, "tc": 1, "auto": 2}[args.engine])
    model = bench_model_device(ctx)
    ctx.set_model(model)
    stream = torch.cuda.current_stream(dev)
    tm = Timed(world, dev, stream)
    peak = fp32_peak(ctx)
    clk = ClockSampler(list(range(world)) if world > 1 else [local_rank])
    csr = args.input == "csr"

    if args.config in ("c2", "c3"):
        head, gen = measure_pipeline(ctx, args.config, args, rank, world, tm, peak, args.steps,
                                     args.warmup, csr=csr, with_e2e=not args.no_e2e, clocks=clk)
        cfg = CONFIGS[args.config]
        stages = None
        if not args.no_stages:
            del gen
            n = head["kernels_per_gpu"]
            dense = ctx.gen_synthetic(n, root=ROOT_SEED, first=rank * n, params=False)
            from paper_2407_13096_b200 import linear_domain
            stages = stage_times(ctx, dense["counts"], dense["dcgm"], cfg,
                                 linear_domain(cfg["nc"], cfg["nm"]), n, stream)
            if csr:
                o = ctx.alloc_pipeline_out(n)
                run_dense = lambda: ctx.pipeline(dense["counts"], dense["dcgm"], cfg["eta"], out=o)  # noqa: E731
                run_dense()  # warm-up: grows the compaction scratch
                stages["pipeline_dense_input_ms"] = cuda_time(stream, run_dense, 3)
            del dense
            if csr:
                stages["realistic_mix"] = realistic_stage(ctx, cfg, stream)
        else:
            del gen
        e2e = head.pop("e2e", None)
        line = {
            "metric": METRIC, "value": head["value"], "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": head["ms_per_step"],
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (gen_kernel stream generated on device; random-init MLP seed 424242)",
            "config": {"workload": cfg["desc"], "kernels_per_gpu": head["kernels_per_gpu"],
                       "grid": head["grid"], "engine": head["engine"], "eta": cfg["eta"],
                       "parallelism": f"kernel-sharded x{world}, no collective",
                       "input": head["input"],
                       "l2": "inputs > 126 MB L2 per step (no flush needed)"},
            "roofline": head["roofline"], "e2e": e2e, "gpu_launches": head["gpu_launches"],
            "clocks": clk.summary(), "stages": stages,
        }
    elif args.config == "c4":
        with clk:
            r = measure_eta(ctx, args, rank, world, tm, peak, args.steps, args.warmup)
        line = {"metric": METRIC, "value": r["value"], "unit": UNIT, "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": r["ms_per_step"],
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
                "data": "synthetic (gen_kernel stream generated on device)",
                "config": {"workload": CONFIGS["c4"]["desc"], "kernels_per_gpu": r["kernels_per_gpu"],
                           "parallelism": f"kernel-sharded x{world}, no collective",
                           "l2": "outputs 3.2 GB per step (> L2)"},
                "roofline": r["roofline"], "triples_per_s": r["triples_per_s"],
                "gpu_launches": r["gpu_launches"], "clocks": clk.summary(), "e2e": None}
    else:  # c5
        with clk:
            r = measure_train(ctx, args, rank, world, tm, peak, args.steps, args.warmup, model)
        line = {"metric": r["metric"], "value": r["value"], "unit": r["unit"], "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": r["ms_per_step"],
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
                "data": "synthetic (gen_kernel stream generated on device)",
                "config": {"workload": CONFIGS["c5"]["desc"], "samples_per_gpu": r["samples_per_gpu"],
                           "batch_per_gpu": r["batch_per_gpu"], "global_batch": r["global_batch"],
                           "parallelism": r["parallelism"],
                           "l2": "batches stream through a 5.6 GB device-resident shard"},
                "roofline": r["roofline"], "gpu_launches": r["gpu_launches"],
                "clocks": clk.summary(), "e2e": None}

    # ---- the other BASELINE configs, measured in the same run (driver-visible) --------
    others = {}
    if not args.no_extra and args.config == "c3":
        ks, kw = max(3, min(args.steps, 10)), 3
        try:
            r, g = measure_pipeline(ctx, "c2", args, rank, world, tm, peak, max(args.steps, 20),
                                    kw, csr=True)
            del g
            others["c2"] = r
            others["c4"] = measure_eta(ctx, args, rank, world, tm, peak, ks, kw)
            others["c5"] = measure_train(ctx, args, rank, world, tm, peak, max(args.steps, 20), kw,
                                         model)
        except Exception as exc:  # reported, never silently dropped
            others["error"] = repr(exc)
        line["configs"] = others
    if rank != 0:
        return
    line["cpu_baseline"] = None
    if not args.no_cpu and world == 1 and args.config in ("c2", "c3"):
        line["cpu_baseline"] = cpu_baseline(args, CONFIGS[args.config], model)
    print(json.dumps(line), flush=True)


def bench_model_device(ctx):
    """bench_model without the CPU oracle: target stats of 65,536 device-generated
    truth parameters (population mean / std)."""
    from paper_2407_13096_b200 import init_mlp
    m = init_mlp(seed=424242)
    p = ctx.gen_synthetic(65536, root=0xC0FFEE, counts=False, dcgm=False)["params"]
    p = p.double().cpu().numpy()
    m.target_mean, m.target_std = p.mean(1), p.std(1)
    return m


def realistic_counts_csr(n, seed=2407, chunk=1 << 19):
    """A realistic PTX category mix, not the generator's fixed 24 slots: every kernel
    lists each of the 126 categories independently with a Zipf-like probability
    (~25 listed categories per kernel, every slot used somewhere), counts log-uniform
    in [1, 2e6].  Returns CSR (row_ptr int64, entries int32 = (count << 7) | slot),
    slot-sorted per kernel."""
    rng = np.random.default_rng(seed)
    w = 1.0 / (1.0 + np.arange(126)) ** 0.8
    w = w[rng.permutation(126)]
    p = np.minimum(w * (25.0 / w.sum()), 0.95)
    rows, ents = [np.zeros(1, np.int64)], []
    total = 0
    for a in range(0, n, chunk):
        m = min(chunk, n - a)
        mask = rng.random((m, 126), dtype=np.float32) < p
        k, sl = np.nonzero(mask)
        cnt = np.exp(rng.random(len(k), dtype=np.float32) * np.float32(np.log(2e6))).astype(np.int64) + 1
        ents.append(((cnt << 7) | sl).astype(np.int32))
        rows.append(total + np.cumsum(mask.sum(1)))
        total += len(k)
    return np.concatenate(rows), np.concatenate(ents)


def realistic_stage(ctx, cfg, stream, n=1 << 22):
    """The CSR pipeline on the realistic mix (4M kernels, same grid / eta), both
    predictor engines, plus the same kernels as dense [126][n] counts."""
    import torch
    rp, ent = realistic_counts_csr(n)
    rp_t, ent_t = torch.from_numpy(rp).cuda(), torch.from_numpy(ent).cuda()
    dcgm = torch.rand((8, n), device="cuda", dtype=torch.float32)
    o = ctx.alloc_pipeline_out(n)
    pairs = cfg["nc"] * cfg["nm"]
    res = {"kernels": n, "nnz_per_kernel": float(len(ent)) / n,
           "slots_used": int(len(np.unique(ent & 127)))}
    for name, eng in (("tc", 1), ("ffma", 0)):
        ctx.set_option("mlp_engine", eng)
        ctx.counters(reset=True)
        ms = cuda_time(stream, lambda: ctx.pipeline_csr(rp_t, ent_t, dcgm, cfg["eta"], out=o), 3)
        c = ctx.counters(reset=True)
        res[f"{name}_ms"] = ms
        res[f"{name}_pairs_per_s"] = n * pairs / (ms * 1e-3)
        if c["tc_tiles"]:
            res["tc_l1_ksteps_per_tile"] = c["tc_l1_ksteps"] / c["tc_tiles"]
    ctx.set_option("mlp_engine", 2)
    dense = torch.zeros((126, n), dtype=torch.int32, device="cuda")
    kk = np.repeat(np.arange(n), np.diff(rp))
    dense[torch.from_numpy(ent & 127).cuda().long(), torch.from_numpy(kk).cuda()] = \
        torch.from_numpy(ent >> 7).cuda()
    res["dense_input_ms"] = cuda_time(stream, lambda: ctx.pipeline(dense, dcgm, cfg["eta"], out=o), 3)
    res["note"] = ("Zipf-like inclusion probabilities over all 126 categories "
                   "(bench.realistic_counts_csr); ms per 4M-kernel call, CUDA events")
    del dense, rp_t, ent_t
    return res


def stage_times(ctx, counts, dcgm, cfg, dom, n, stream):
    import torch
    fused = ctx.featurize(counts, dcgm)
    params, _, _ = ctx.predict_params(fused)
    res = {}

    def t(fn, reps=3):
        fn()
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(reps):
            fn()
        b.record(stream)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / reps

    res["featurize_ms"] = t(lambda: ctx.featurize(counts, dcgm, out=fused))
    res["featurize_gbs"] = n * 1072 / (res["featurize_ms"] * 1e-3) / 1e9
    res["predict_ms"] = t(lambda: ctx.predict_params(fused))
    res["predict_tflops"] = n * MLP_FLOPS / (res["predict_ms"] * 1e-3) / 1e12
    res["sweep_ms"] = t(lambda: ctx.brute_force_config(params, cfg["eta"]))
    res["sweep_pairs_per_s"] = n * dom.pairs / (res["sweep_ms"] * 1e-3)
    res["sweep_tflops"] = res["sweep_pairs_per_s"] * PAIR_FLOPS / 1e12
    p64 = params[:, : min(n, 1 << 22)].double().t().contiguous()
    res["sweep_f64_ms_4M"] = t(lambda: ctx.brute_force_config_exact(p64, cfg["eta"]))
    res["sweep_f64_pairs_per_s"] = p64.shape[0] * dom.pairs / (res["sweep_f64_ms_4M"] * 1e-3)
    res["optimal_config_ms_4M"] = t(lambda: ctx.optimal_config(p64, cfg["eta"]))
    res["optimal_config_kernels_per_s"] = p64.shape[0] / (res["optimal_config_ms_4M"] * 1e-3)
    # param_fit: 1M kernels measured on the reference's default 14x3 grid (run_campaign)
    nf = min(n, 1 << 20)
    core = [705.0 + 52.0 * k for k in range(13)] + [1380.0]
    grid = []
    for fc in core:
        d = fc / 1000.0 - 0.5
        for fm in (438.0, 658.0, 877.0):
            grid.append([2.0 * d * d + 0.5, fc, fm])
    g = torch.tensor(grid, dtype=torch.float64, device=params.device)
    pp = p64[:nf].t()  # [7, nf]
    vc, fc, fm = g[:, 0:1], g[:, 1:2], g[:, 2:3]
    P = ((pp[0] + pp[1] * vc) + pp[2] * fm) + ((pp[3] * vc) * vc) * fc      # [42, nf]
    T = pp[4] + torch.maximum(pp[5] / fm, pp[6] / fc)
    P, T = P.contiguous(), T.contiguous()
    res["param_fit_ms_1M"] = t(lambda: ctx.param_fit(grid, P, T))
    res["param_fit_kernels_per_s"] = nf / (res["param_fit_ms_1M"] * 1e-3)
    del fused, params, p64, P, T
    return res


def cpu_baseline(args, cfg, model):
    import oracle
    port = oracle.port()
    try:
        ref = oracle.ref()
    except (FileNotFoundError, OSError):
        ref = None
    threads = oracle.oracle.default_threads()
    n = args.cpu_sample or 131072
    rate, secs, det = cpu_pipeline_rate(port, ref, n, cfg, model, threads)
    return {"value": rate, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": (f"{n} kernels of the {args.config} workload, {secs:.1f} s on {threads} "
                       f"threads; features+MLP: C restatement (reference needs Eigen, absent), "
                       f"{det['features_mlp_s']:.2f} s; sweep: {det['sweep_impl']}, "
                       f"{det['sweep_s']:.2f} s")}


def self_launch(args):
    """`--gpus N` without a launcher: start N ranks of this script on this node (one
    process per GPU), with the torchrun environment (RANK, LOCAL_RANK, WORLD_SIZE,
    MASTER_ADDR=127.0.0.1, MASTER_PORT) and NCCL_DEBUG=INFO so NCCL's communicator
    lines (nranks) land in stderr.  Returns the worst exit code."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    procs = []
    for r in range(args.gpus):
        env = dict(os.environ, RANK=str(r), LOCAL_RANK=str(r), WORLD_SIZE=str(args.gpus),
                   LOCAL_WORLD_SIZE=str(args.gpus), MASTER_ADDR="127.0.0.1",
                   MASTER_PORT=str(port))
        env.setdefault("NCCL_DEBUG", "INFO")
        procs.append(subprocess.Popen([sys.executable, os.path.abspath(__file__)] + sys.argv[1:],
                                      env=env))
    return max(p.wait() for p in procs)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(self_launch(args))
    world = env_int("WORLD_SIZE", 1)
    rank = env_int("RANK", 0)
    local_rank = env_int("LOCAL_RANK", 0)
    if world > 1:
        import torch
        import torch.distributed as dist
        if args.impl == "ours":
            torch.cuda.set_device(local_rank)
            os.environ.setdefault("NCCL_DEBUG", "INFO")
        dist.init_process_group("nccl" if args.impl == "ours" else "gloo")
    try:
        if args.impl == "reference":
            run_reference(args, rank, world)
        else:
            run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
