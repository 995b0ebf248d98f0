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
def cpu_pipeline_rate(port, ref, n, cfg, model, threads):
    """Host-CPU reference path on n kernels: features + MLP (C restatement; the
    reference needs Eigen, absent) and brute_force_config (the reference's own
    optimizer.cpp, oracle/_ref).  Returns (pairs/s, seconds, detail)."""
    from paper_2407_13096_b200 import linear_domain
    dom = linear_domain(cfg["nc"], cfg["nm"])
    dev = dom.dev.as_array()
    g = port.gen_stream(ROOT_SEED, n, want=("counts", "dcgm"), threads=threads)
    t0 = time.perf_counter()
    fused = port.fuse(g["counts"], g["dcgm"])
    params, _ = port.predict_params(model, fused, threads=threads)
    t1 = time.perf_counter()
    eta = cfg["eta"] if cfg["eta"] is not None else 0.8
    if ref is not None:
        ref.brute_force_config(params, dom.core_freqs_mhz, dom.mem_freqs_mhz, dev, eta,
                               dom.dev.pmax_w, threads=threads)
        sweep_kind = "reference optimizer.cpp (oracle/_ref)"
    else:
        port.brute_force(params, dom.core_freqs_mhz, dom.mem_freqs_mhz, dev, eta,
                         dom.dev.pmax_w, threads=threads)
        sweep_kind = "C restatement (oracle/liboracle.so)"
    t2 = time.perf_counter()
    pairs = n * dom.pairs
    return pairs / (t2 - t0), t2 - t0, {"features_mlp_s": t1 - t0, "sweep_s": t2 - t1,
                                         "sweep_impl": sweep_kind}


def bench_model(port=None):
    """Model for the benchmark: Glorot init (seed 424242, the golden seed) with
    target stats of the synthetic truth parameters so outputs are DVFS-scaled."""
    from paper_2407_13096_b200 import init_mlp
    m = init_mlp(seed=424242)
    # population mean / std of the generator's parameter ranges, from 65,536 draws
    if port is not None:
        p = port.gen_stream(0xC0FFEE, 65536, want=("params",))["params"]
        m.target_mean, m.target_std = p.mean(0), p.std(0)
    return m


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
def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    from paper_2407_13096_b200 import linear_domain
    from paper_2407_13096_b200.api import Context, _ptr
    from paper_2407_13096_b200 import _lib

    cfg = CONFIGS[args.config]
    n = args.kernels or cfg["n"]
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    dom = linear_domain(cfg["nc"], cfg["nm"])
    ctx = Context(local_rank)
    ctx.set_option("mlp_engine", {"ffma": 0, "tc": 1, "auto": 2}[args.engine])
    ctx.set_domain(dom)
    model = bench_model_device(ctx)
    ctx.set_model(model)
    stream = torch.cuda.current_stream(dev)

    if args.config == "c5":
        return run_train(args, rank, world, local_rank, ctx, dom, model, n)
    # inputs: this rank's shard [rank*n, (rank+1)*n) of the global synthetic stream
    csr = args.input == "csr" and args.config != "c4"
    if csr:
        gen = ctx.gen_synthetic_csr(n, root=ROOT_SEED, first=rank * n)
        counts = None
        dcgm = gen["dcgm"]
    else:
        gen = ctx.gen_synthetic(n, root=ROOT_SEED, first=rank * n, params=(args.config == "c4"))
        counts, dcgm = gen["counts"], gen["dcgm"]
    etas = np.arange(101) / 100.0
    if args.config == "c4":
        params = gen["params"]
        idx_o = torch.empty((101, n), dtype=torch.int32, device=dev)
        cost_o = torch.empty((101, n), dtype=torch.float32, device=dev)
        eta_arr = np.ascontiguousarray(etas)
        dp = __import__("ctypes").POINTER(__import__("ctypes").c_double)

        def step():
            ctx._raise(ctx._lib.dso_eta_sweep(ctx._h, _ptr(params), n, n,
                                              eta_arr.ctypes.data_as(dp), 101, dom.dev.pmax_w,
                                              _ptr(idx_o), _ptr(cost_o), n))
        units_per_step = n * dom.pairs  # (kernel, pair) evals; x101 etas reported separately
        flops_per_step = n * dom.pairs * (9 + 3 * 101)  # P,T,E once + 3 per (pair, eta)
    else:
        out = ctx.alloc_pipeline_out(n)
        if csr:
            def step():
                ctx.pipeline_csr(gen["row_ptr"], gen["entries"], dcgm, cfg["eta"], out=out)
        else:
            def step():
                ctx.pipeline(counts, dcgm, cfg["eta"], out=out)
        units_per_step = n * dom.pairs
        flops_per_step = n * (MLP_FLOPS + PAIR_FLOPS * dom.pairs)
        if csr:
            # Sparse input: layer 1 only needs the rows a kernel lists (8 DCGM rows +
            # its non-zero count slots; the kernel skips all-zero rows exactly), so
            # the algorithmic work is 2*100*(8 + nnz) there, not 2*100*134.
            nnz = float((gen["row_ptr"][n] - gen["row_ptr"][0]).item()) / n
            flops_per_step = n * (mlp_flops_sparse(8 + nnz) + PAIR_FLOPS * dom.pairs)

    # measured FP32 peak (roofline denominator for the FP32-pipe-bound kernels)
    peak = {}
    for mode, name in ((1, "ffma2"), (0, "ffma")):
        v = __import__("ctypes").c_double()
        ctx._raise(_lib.lib().dso_probe_fp32_peak(ctx._h, mode, __import__("ctypes").byref(v)))
        peak[name] = v.value

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    barrier()
    launches0 = ctx.launch_count
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(list(range(world)) if world > 1 else [local_rank]) as clk:
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
    barrier()
    launches = ctx.launch_count - launches0
    ms = e0.elapsed_time(e1) / args.steps
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    value = units_per_step * world / (ms_max * 1e-3)

    # ---- per-stage breakdown (same data, separate kernels) ---------------------------
    stages = None
    if not args.no_stages and args.config != "c4":
        dense = ctx.gen_synthetic(n, root=ROOT_SEED, first=rank * n, params=False)
        stages = stage_times(ctx, dense["counts"], dense["dcgm"], cfg, dom, n, stream)
        if csr:
            a = torch.cuda.Event(enable_timing=True)
            bb = torch.cuda.Event(enable_timing=True)
            ctx.pipeline(dense["counts"], dense["dcgm"], cfg["eta"], out=out)
            a.record(stream)
            for _ in range(3):
                ctx.pipeline(dense["counts"], dense["dcgm"], cfg["eta"], out=out)
            bb.record(stream)
            torch.cuda.synchronize()
            stages["pipeline_dense_input_ms"] = a.elapsed_time(bb) / 3
        del dense

    # ---- end to end through the C-ABI with pinned host buffers --------------------------
    e2e = None
    if not args.no_e2e and args.config != "c4":
        hd = dcgm.cpu().pin_memory()
        if csr:
            hrp = gen["row_ptr"].cpu().pin_memory()
            hent = gen["entries"].cpu().pin_memory()
            h2d = (n + 1) * 8 + hent.numel() * 4 + n * 8 * 4
            run_e2e = lambda o: ctx.pipeline_csr(hrp, hent, hd, cfg["eta"], out=o)  # noqa: E731
        else:
            hc = counts.cpu().pin_memory()
            h2d = n * (126 * 4 + 8 * 4)
            run_e2e = lambda o: ctx.pipeline(hc, hd, cfg["eta"], out=o)  # noqa: E731
        hout = ctx.alloc_pipeline_out(n, host=True, like=hd)
        run_e2e(hout)  # warm-up (staging buffers)
        k = max(1, min(args.steps, 5))
        barrier()
        t0 = time.perf_counter()
        for _ in range(k):
            run_e2e(hout)
        el = (time.perf_counter() - t0) / k
        te = torch.tensor([el], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        el = float(te.item())
        e2e = {"value": units_per_step * world / el, "unit": UNIT,
               "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(n * 16), "ms_per_step": el * 1e3,
               "steps": k, "timing": "host wall clock around synchronous C-ABI calls "
                                     "(dso_pipeline%s with DSO_HOST, pinned buffers)"
                                     % ("_csr" if csr else "")}
        del hd, hout

    if rank != 0:
        return
    achieved = flops_per_step / (ms * 1e-3) / 1e12
    peaks = measured_peaks()
    pk = peak["ffma2"]
    # which predictor engine ran (the library's auto policy: tcgen05 for CSR input)
    engine_used = ("tc" if args.config != "c4" and (args.engine == "tc" or
                                                      (args.engine == "auto" and csr))
                   else ("ffma" if args.config != "c4" else None))
    roofline = {
        "bound": "fp32", "achieved": achieved, "peak": pk, "unit": "TFLOP/s",
        "frac": achieved / pk,
        "traffic": ncu_traffic(args.config, n) if (csr or args.config == "c4") else None,
        "traffic_unit": "bytes per launch (ncu dram__bytes_read+write, profiles/ncu_summary.json)",
        "algorithmic_bytes_per_launch": (n * ((136 if csr else 536) + 16) if args.config != "c4"
                                         else n * (28 + 101 * 8)),
        "kernel": "ws_kernel (fused pipeline)" if args.config != "c4" else "eta_sweep_fast_kernel",
        "flops_per_kernel": flops_per_step / n if args.config != "c4" else None,
        "flops_note": ("layer 1 counted on the 8 DCGM + non-zero count rows of each kernel "
                       "(CSR input; all-zero rows are skipped exactly); the dense-input "
                       "count (SURVEY.md §8(d): 39,650 + 14 per pair) is "
                       "flops_per_kernel_dense" if csr and args.config != "c4" else
                       ("9 flops per (kernel, pair) for P, T, E plus 3 per (kernel, pair, eta); "
                        "the kernel is bound by the ALU pipe (group min trees and selects: "
                        "profiles/r1/ncu_eta_sweep_metrics.txt)" if args.config == "c4" else None)),
        "flops_per_kernel_dense": (MLP_FLOPS + PAIR_FLOPS * dom.pairs)
        if args.config != "c4" else None,
        "peak_source": ("measured in this run by dso_probe_fp32_peak (FFMA2 loop, 148x4 CTAs); "
                        "MEASURED_PEAKS.json has no FP32 figure"),
        "peak_ffma_scalar": peak["ffma"],
        "nominal_peak": 148 * 128 * 2 * peaks.get("sm_max_mhz", 1965.0) * 1e6 / 1e12,
        "hbm_gbs_measured": peaks.get("hbm_gbs"),
        "achieved_input_gbs": (n * (136 if csr else 536) / (ms * 1e-3) / 1e9
                               if args.config != "c4" else None),
    }
    if engine_used == "tc":
        # the tcgen05 engine: layers 1-2 as 3xTF32 MMAs (3 TF32 products per
        # multiply-add), layers 3-4 and the sweep on the FMA pipe; roofline against
        # the dense TF32 tensor peak (half the measured dense bf16 figure)
        tc_flops = n * 3 * 2 * (134 * 100 + 100 * 50)
        tc_peak = peaks.get("bf16_tflops", 2250.0) / 2
        fp32_view = dict(roofline)
        roofline = {
            "bound": "tensor", "achieved": tc_flops / (ms * 1e-3) / 1e12, "peak": tc_peak,
            "unit": "TFLOP/s", "frac": tc_flops / (ms * 1e-3) / 1e12 / tc_peak,
            "traffic": fp32_view["traffic"], "traffic_unit": fp32_view["traffic_unit"],
            "algorithmic_bytes_per_launch": fp32_view["algorithmic_bytes_per_launch"],
            "kernel": "tc_kernel (fused pipeline, tcgen05 kind::tf32)",
            "tensor_flops_per_kernel": 3 * 2 * (134 * 100 + 100 * 50),
            "flops_note": "TF32 tensor products issued for layers 1-2 (3xTF32: hi.hi + hi.lo + "
                          "lo.hi per multiply-add, dense K = 134 / 100); CSR tiles skip all-zero "
                          "8-column chunks of layer 1, so the issued count is lower than this",
            "peak_source": "MEASURED_PEAKS.json bf16_tflops / 2 (dense TF32 = half the bf16 rate)",
            "fp32_equivalent": {"achieved": achieved, "peak": pk, "frac": achieved / pk,
                                "flops_per_kernel": fp32_view["flops_per_kernel"]},
            "hbm_gbs_measured": peaks.get("hbm_gbs"),
            "achieved_input_gbs": fp32_view["achieved_input_gbs"],
        }
    cpu = None
    if not args.no_cpu and world == 1:
        cpu = cpu_baseline(args, cfg, model)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (gen_kernel stream generated on device; random-init MLP seed 424242)",
        "config": {"workload": cfg["desc"], "kernels_per_gpu": n, "grid": f"{cfg['nc']}x{cfg['nm']}",
                   "engine": engine_used or args.engine,
                   "eta": cfg["eta"] if cfg["eta"] is not None else "0.00..1.00 (101)",
                   "parallelism": f"kernel-sharded x{world}, no collective",
                   "input": ("sparse per-kernel PTX count lists (24 non-zeros/kernel) + DCGM"
                             if csr else "dense [126][n] PTX counts + DCGM"),
                   "l2": "inputs > 126 MB L2 per step (no flush needed)"},
        "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
        "clocks": clk.summary(), "stages": stages,
    }
    if args.config == "c4":
        line["triples_per_s"] = value * 101
    print(json.dumps(line), flush=True)


def run_train(args, rank, world, local_rank, ctx, dom, model, n):
    """C5: synchronous data-parallel SGD steps (device grad -> NCCL allreduce ->
    device update) over a device-resident 10M-sample shard per GPU."""
    import torch
    import torch.distributed as dist

    from paper_2407_13096_b200.train import DataParallelTrainer
    cfg = CONFIGS["c5"]
    dev = torch.device("cuda", local_rank)
    stream = torch.cuda.current_stream(dev)
    B = cfg["batch"]
    gen = ctx.gen_synthetic(n, root=0xACCE5505, first=rank * n)
    x = ctx.featurize(gen["counts"], gen["dcgm"])
    del gen["counts"]
    p = gen["params"].double()
    mean = torch.tensor(model.target_mean, dtype=torch.float64, device=dev)
    std = torch.tensor(model.target_std, dtype=torch.float64, device=dev)
    y = ((p - mean[:, None]) / std[:, None]).float().contiguous()
    del p, gen
    tr = DataParallelTrainer(ctx, lr=0.1)
    nb = n // B
    grad = torch.empty((ctx.n_model_params,), dtype=torch.float32, device=dev)

    def step(i):
        s = (i % nb) * B
        g, loss = ctx.train_grad_slice(x, y, s, B, grad=grad)
        tr.allreduce(g)
        tr.allreduce(loss)
        ctx.train_apply(g, tr.lr, 1.0 / (B * world * 7))
        return loss

    def barrier():
        if world > 1:
            dist.barrier()

    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()
    barrier()
    launches0 = ctx.launch_count
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(list(range(world)) if world > 1 else [local_rank]) as clk:
        e0.record(stream)
        for i in range(args.steps):
            step(args.warmup + i)
        e1.record(stream)
        torch.cuda.synchronize()
    barrier()
    ms = e0.elapsed_time(e1) / args.steps
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    # grad kernel alone (share of the step)
    a = torch.cuda.Event(enable_timing=True)
    bb = torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for i in range(5):
        ctx.train_grad_slice(x, y, (i % nb) * B, B, grad=grad)
    bb.record(stream)
    torch.cuda.synchronize()
    grad_ms = a.elapsed_time(bb) / 5
    if rank != 0:
        return
    value = B * world / (ms_max * 1e-3)
    achieved = B * TRAIN_FLOPS / (grad_ms * 1e-3) / 1e12
    v = __import__("ctypes").c_double()
    from paper_2407_13096_b200 import _lib
    ctx._raise(_lib.lib().dso_probe_fp32_peak(ctx._h, 1, __import__("ctypes").byref(v)))
    line = {
        "metric": "predictor training sample-steps/s (C5)", "value": value,
        "unit": "samples/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_max, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (gen_kernel stream generated on device)",
        "config": {"workload": cfg["desc"], "samples_per_gpu": n, "batch_per_gpu": B,
                   "global_batch": B * world, "parallelism": f"dp{world} (NCCL allreduce)"},
        "roofline": {"bound": "fp32", "achieved": achieved, "peak": v.value, "unit": "TFLOP/s",
                     "frac": achieved / v.value, "traffic": ncu_traffic("c5", B),
                     "traffic_unit": "bytes per dso_train_grad (ncu, profiles/ncu_summary.json)",
                     "kernel": "train_fb_kernel + train_wgrad_kernel + reduce_partials",
                     "flops_per_sample": TRAIN_FLOPS, "grad_kernel_ms": grad_ms},
        "gpu_launches": ctx.launch_count - launches0, "clocks": clk.summary(),
    }
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


def main():
    args = parse()
    world = env_int("WORLD_SIZE", 1)
    rank = env_int("RANK", 0)
    local_rank = env_int("LOCAL_RANK", 0)
    if world > 1:
        import torch
        import torch.distributed as dist
        if args.impl == "ours":
            torch.cuda.set_device(local_rank)
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
