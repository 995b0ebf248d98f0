"""Copy the judged evidence of a gpurun session into profiles/ (tracked).

usage: python scripts/summarize_profiles.py gpurun_out/<tag> profiles/<round>
Writes: ncu key metrics of the captured kernel, the per-kernel launch summary,
the bench JSON lines, and profiles/ncu_summary.json (DRAM traffic per kernel of
the dominant launch, read by bench.py for roofline.traffic)."""
import csv
import io
import json
import os
import shutil
import subprocess
import sys
from collections import defaultdict

src, dst = sys.argv[1], sys.argv[2]
os.makedirs(dst, exist_ok=True)
KEYS = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smsp__inst_executed.sum",
        "launch__registers_per_thread", "launch__block_size", "launch__grid_size",
        "launch__shared_mem_per_block_dynamic",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"]
summary = {}
def dump_metrics(rep, out):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    if len(rows) < 3:
        return None, None
    hdr, units, vals = rows[0], rows[1], rows[2]
    d, u = dict(zip(hdr, vals)), dict(zip(hdr, units))
    with open(out, "w") as f:
        f.write(f"# ncu --set full --clock-control none capture of {rep}\n")
        for k in KEYS:
            if k in d:
                f.write(f"{k}\t{d.get(k)}\t{u.get(k, '')}\n")
    return d, u


# the FMA-pipe engine's kernel on the same workload (bench --engine ffma)
rp = os.path.join(src, "prof_pipeline_ffma.ncu-rep")
if os.path.exists(rp):
    dump_metrics(rp, os.path.join(dst, "ncu_ws_kernel_ffma_metrics.txt"))
rep = os.path.join(src, "prof_pipeline.ncu-rep")
if os.path.exists(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = dict(zip(hdr, vals))
    u = dict(zip(hdr, units))
    with open(os.path.join(dst, "ncu_c3_kernel_metrics.txt"), "w") as f:
        f.write(f"# ncu --set full --clock-control none capture of {rep}\n")
        for k in KEYS:
            f.write(f"{k}\t{d.get(k)}\t{u.get(k, '')}\n")
    log = open(os.path.join(src, "ncu_full.log")).read()
    n_kernels = 2097152
    mb = float(d["dram__bytes_read.sum"]) + float(d["dram__bytes_write.sum"])
    scale = 1e6 if u.get("dram__bytes_read.sum", "").startswith("M") else 1e9
    summary["c3"] = {"kernel": d["Kernel Name"], "kernels_per_launch": n_kernels,
                     "dram_bytes_per_launch": mb * scale,
                     "dram_bytes_per_kernel": mb * scale / n_kernels,
                     "source": f"{dst}/ncu_c3_kernel_metrics.txt (ncu --set full, "
                               f"{n_kernels} kernels, CSR input)"}
    lines = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                            "cuda,sass"], capture_output=True, text=True).stdout
    with open(os.path.join(dst, "ncu_c3_kernel_source_hot_lines.txt"), "w") as f:
        out = subprocess.run([sys.executable, "scripts/ncu_lines.py", rep, "40"],
                             capture_output=True, text=True).stdout
        f.write(out)
# secondary kernels: eta sweep (C4) and training (C5) key metrics
for rep_name, tag in (("prof_eta.ncu-rep", "eta_sweep"), ("prof_train.ncu-rep", "train")):
    rp = os.path.join(src, rep_name)
    if not os.path.exists(rp):
        continue
    txt = subprocess.run(["ncu", "-i", rp, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    with open(os.path.join(dst, f"ncu_{tag}_metrics.txt"), "w") as f:
        f.write(f"# ncu --set full --clock-control none capture of {rp}\n")
        for vals in rows[2:]:
            d = dict(zip(rows[0], vals))
            u = dict(zip(rows[0], rows[1]))
            f.write(f"## {d.get('Kernel Name')}\n")
            for k in KEYS[1:]:
                f.write(f"{k}\t{d.get(k)}\t{u.get(k, '')}\n")
# DRAM traffic per unit for the C4 (eta sweep, 1M-kernel capture) and C5 (training,
# 65,536-sample batch: the forward/backward + weight-gradient kernels) roofline lines
for rep_name, cfg_key, units, unit_name in (("prof_eta.ncu-rep", "c4", 1048576, "kernel"),
                                            ("prof_train.ncu-rep", "c5", 65536, "sample")):
    rp = os.path.join(src, rep_name)
    if not os.path.exists(rp):
        continue
    txt = subprocess.run(["ncu", "-i", rp, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    tot, names = 0.0, []
    for vals in rows[2:]:
        d = dict(zip(rows[0], vals))
        u = dict(zip(rows[0], rows[1]))
        sc = 1e6 if u.get("dram__bytes_read.sum", "").startswith("M") else (
            1e9 if u.get("dram__bytes_read.sum", "").startswith("G") else 1e3)
        tot += (float(d["dram__bytes_read.sum"]) + float(d["dram__bytes_write.sum"])) * sc
        names.append(d["Kernel Name"].split("(")[0])
    summary[cfg_key] = {"kernel": " + ".join(names), "units_per_capture": units,
                        f"dram_bytes_per_{unit_name}": tot / units,
                        "dram_bytes_per_kernel": tot / units,
                        "source": f"{dst}/ncu_{'eta_sweep' if cfg_key == 'c4' else 'train'}"
                                  f"_metrics.txt (ncu --set full)"}
for extra in ("phase_timing.txt", "launches_c5.csv"):
    p = os.path.join(src, extra)
    if os.path.exists(p):
        shutil.copy(p, os.path.join(dst, extra))
lc = os.path.join(src, "launches.csv")
if os.path.exists(lc):
    rows = list(csv.reader(open(lc)))
    st = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[st]
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[st + 1:]:
        d = dict(zip(hdr, r))
        name = d["Kernel Name"].split("(")[0].replace("dso_b200::<unnamed>::", "")
        agg[name][0] += 1
        agg[name][1] += float(d["Metric Value"])
    with open(os.path.join(dst, "launch_list_summary.txt"), "w") as f:
        f.write("# ncu --metrics gpu__time_duration.sum --clock-control none, bench.py --steps 2 "
                "--warmup 1 --kernels 4194304 (cold-cache, serialised: compare shares)\n")
        f.write("launches\ttotal_ms\tkernel\n")
        for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
            f.write(f"{c}\t{t / 1e6:.3f}\t{k}\n")
    shutil.copy(lc, os.path.join(dst, "launches.csv"))
for name in ("bench", "bench_ref", "bench_c2", "bench_c4", "bench_c5", "bench_ffma", "bench_dense"):
    p = os.path.join(src, name + ".log")
    if os.path.exists(p):
        for line in open(p):
            if line.startswith("{"):
                open(os.path.join(dst, name + ".json"), "w").write(line.strip() + "\n")
                break
for extra in ("pytest_gpu.log", "memcheck.log", "racecheck.log", "synccheck.log", "smoke.log",
              "nvidia-smi.txt", "nproc.txt", "tc_phase.txt", "phase_timing.txt"):
    p = os.path.join(src, extra)
    if os.path.exists(p):
        shutil.copy(p, os.path.join(dst, extra))
if summary:
    path = os.path.join("profiles", "ncu_summary.json")
    old = json.load(open(path)) if os.path.exists(path) else {}
    old.update(summary)
    json.dump(old, open(path, "w"), indent=1)
print("wrote", sorted(os.listdir(dst)))
