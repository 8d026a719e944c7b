"""Write the round's ncu evidence under profiles/ from gpurun_out/<dir>/ (run here, no GPU needed).
    python tools/summarize_profiles.py r02 gpurun_out/r2

Inputs (tools/bench_round.sh): launches.csv (ncu launch list of a short default bench) and
prof_<name>.ncu-rep (ncu --set full, one launch each).  Outputs: profiles/launches_<tag>.csv,
profiles/ncu_summary_<tag>.md and profiles/ncu_traffic.json (per-launch DRAM bytes of the SV kernel
at the bench's launch size, read by bench.py's roofline "traffic")."""
import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")
UNITS = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}

# name -> (what one captured launch processes, algorithmic bytes or flops of it, the bench's launch scale)
KERNELS = {
    "loss_sv": dict(title="loss_sv_kernel: fused fwd+bwd, 16,384 rows x 151,936 bf16 columns (tools/kbench.py)",
                    rows=16384, bytes_per_row=2 * 151936 * 2 + 17, bench_rows=131072),
    "vpcache8": dict(title="vp_cache_kernel<6,3>: one rank's shard at P = 8, 65,536 rows x 18,992 columns "
                           "(tools/vpbench.py --peer)", rows=65536, bytes_per_row=2 * 18992 * 2 + 17, bench_rows=65536),
    "vpcache4": dict(title="vp_cache_kernel<11,2>: one rank's shard at P = 4, 65,536 rows x 37,984 columns",
                     rows=65536, bytes_per_row=2 * 37984 * 2 + 17, bench_rows=65536),
    "ring4": dict(title="vp_ring_kernel (L2 re-read, D = 3, 5-vector slots, two service warps): one rank's shard "
                        "at P = 4, 65,536 rows x 37,984 columns (tools/vpbench.py --peer --ring; the default "
                        "across 4 GPUs)",
                  rows=65536, bytes_per_row=2 * 37984 * 2 + 17, bench_rows=65536),
    "ring2": dict(title="vp_ring_kernel (L2 re-read, D = 1, two service warps): one rank's shard at P = 2, "
                        "65,536 rows x 75,968 columns (the default across 2 GPUs)",
                  rows=65536, bytes_per_row=2 * 75968 * 2 + 17, bench_rows=65536),
    "lmgrad": dict(title="lmhead_kernel<grad>: logits recompute + G = s (p - onehot), 8,192 tokens x d 4,096 x "
                         "V 151,936 (one backward chunk of tools/lmbench.py --bwd)", tokens=8192, d=4096, V=151936),
    "lmfwd": dict(title="lmhead_kernel<logprob>: 16,384 tokens x d 4,096 x V 151,936 (tools/lmbench.py)",
                  tokens=16384, d=4096, V=151936),
}


def _base(name):
    """'void rl::loss_sv_kernel<bf16_t, 2>(rl::ClArgs)' -> 'loss_sv_kernel'"""
    n = name.split("(")[0].replace("void ", "").split("<")[0]
    return n.split("::")[-1].strip()


def _library_kernels():
    """__global__ function names defined in the library's sources"""
    import glob
    import re
    names = set()
    for f in glob.glob(os.path.join(ROOT, "paper_2605_15565_b200", "csrc", "*.cu")):
        names |= set(re.findall(r"__global__\s+void\s+(?:__launch_bounds__\([^)]*\)\s+)?(\w+)\s*\(", open(f).read()))
    return names


def launches(src, tag):
    rows = list(csv.reader(open(os.path.join(src, "launches.csv"))))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h, data = rows[hi], rows[hi + 1:]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    timed = [r for r in data if len(r) > vi and r[mi] == "gpu__time_duration.sum"]
    n_all = len(timed)
    ours = [(r[ki], float(r[vi].replace(",", ""))) for r in timed if _base(r[ki]) in _library_kernels()]
    with open(os.path.join(PROF, f"launches_{tag}.csv"), "w") as f:
        f.write("# ncu --nvtx --nvtx-include timed/ --metrics gpu__time_duration.sum --clock-control none, command: "
                "python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu (the timed region only; cold-cache, "
                "serialised launches: compare shares)\n")
        f.write(f"# launches in the timed region: {n_all}, of this library: {len(ours)}\nkernel,ns\n")
        for k, v in ours:
            f.write(f"\"{k[:90]}\",{v:.0f}\n")
    agg = collections.defaultdict(list)
    for k, v in ours:
        agg[k.split("(")[0].replace("void ", "").replace("rl::", "")[:70]].append(v)
    tot = sum(sum(v) for v in agg.values())
    lines = [f"launches in bench.py's timed region (ncu --nvtx-include timed/): {n_all}, of this library: "
             f"{len(ours)}", f"{'kernel':72s} {'n':>5s} {'avg_us':>10s} {'share':>7s}"]
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"{k:72s} {len(v):5d} {sum(v) / len(v) / 1e3:10.1f} {100 * sum(v) / tot:6.2f}%")
    return "\n".join(lines)


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    return dict(zip(r[0], r[2])), dict(zip(r[0], r[1]))


def main():
    tag, src = sys.argv[1], sys.argv[2]
    os.makedirs(PROF, exist_ok=True)
    summary = [f"# ncu evidence, round {tag} (source: {src}; builder-run, B200, --clock-control none)", "",
               "## Launch list of bench.py (our kernels)", "```", launches(src, tag), "```", ""]
    traffic = {}
    for name, kd in KERNELS.items():
        p = os.path.join(src, f"prof_{name}.ncu-rep")
        if not os.path.exists(p):
            continue
        d, units = raw(p)

        def g(k):
            try:
                return float(d[k].replace(",", "")) * UNITS.get(units.get(k, ""), 1.0)
            except (KeyError, ValueError):
                return float("nan")
        rd, wr = g("dram__bytes_read.sum"), g("dram__bytes_write.sum")
        summary += [f"## {name}: {kd['title']}", "```"]
        for k in ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
                  "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
                  "sm__throughput.avg.pct_of_peak_sustained_elapsed",
                  "smsp__issue_active.avg.pct_of_peak_sustained_active",
                  "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
                  "sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active",
                  "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
                  "lts__t_sector_hit_rate.pct", "launch__registers_per_thread", "launch__grid_size",
                  "launch__block_size", "launch__cluster_dim_x", "sm__ctas_launched.sum"]:
            if k in d:
                summary.append(f"{k:62s} {d[k]} {units.get(k, '')}")
        if "rows" in kd:
            alg = kd["bytes_per_row"]
            per_row = (rd + wr) / kd["rows"]
            summary.append(f"{'algorithmic bytes per row':62s} {alg}")
            summary.append(f"{'dram bytes per row (measured)':62s} {per_row:.0f}  ({per_row / alg:.4f} x algorithmic)")
            traffic[name] = {"dram_bytes_per_launch": per_row * kd["bench_rows"], "dram_bytes_per_row": per_row,
                             "algorithmic_bytes_per_row": alg, "captured_rows": kd["rows"], "read_bytes": rd,
                             "write_bytes": wr, "note": f"ncu --set full of a {kd['rows']}-row launch; per-launch "
                                                        f"figure scaled to the bench's {kd['bench_rows']}-row launch"}
        else:
            ops = (kd["tokens"] + kd["V"]) * kd["d"] * 2
            flops = 2.0 * kd["tokens"] * kd["V"] * kd["d"]
            t = g("gpu__time_duration.sum") / 1e9 if units.get("gpu__time_duration.sum") == "ns" else \
                float(d["gpu__time_duration.sum"].replace(",", "")) * {"usecond": 1e-6, "msecond": 1e-3}.get(
                    units.get("gpu__time_duration.sum", "msecond"), 1e-3)
            summary.append(f"{'operand bytes (h + W, bf16)':62s} {ops:.3e}")
            summary.append(f"{'dram read / operand bytes':62s} {rd / ops:.3f}")
            summary.append(f"{'dram write bytes':62s} {wr:.3e}"
                           + (f"  (G written: {kd['tokens'] * kd['V'] * 2:.3e})" if name == "lmgrad" else ""))
            summary.append(f"{'TFLOP/s (2 N V d / duration, under ncu)':62s} {flops / t / 1e12:.1f}")
        st = sorted(((k, g(k)) for k in d if k.startswith("smsp__pcsamp_warps_issue_stalled")
                     and not k.endswith("not_issued")), key=lambda kv: -kv[1])
        tot = sum(v for _, v in st if v == v)
        summary.append("stall reasons (pc sampling):")
        for k, v in st[:8]:
            summary.append(f"   {k.replace('smsp__pcsamp_warps_issue_stalled_', ''):28s} {100 * v / tot:6.2f}%")
        summary += ["```", ""]
    if "loss_sv" in traffic:
        traffic["sv"] = traffic["loss_sv"]   # the key bench.py reads
    with open(os.path.join(PROF, "ncu_traffic.json"), "w") as f:
        json.dump(traffic, f, indent=1)
    with open(os.path.join(PROF, f"ncu_summary_{tag}.md"), "w") as f:
        f.write("\n".join(summary) + "\n")
    print("\n".join(summary))


if __name__ == "__main__":
    main()
