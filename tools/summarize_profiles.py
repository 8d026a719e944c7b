"""Write the round's ncu evidence under profiles/ from gpurun_out/ (run here, no GPU needed).
    python tools/summarize_profiles.py r01"""
import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")


def launches(tag):
    rows = list(csv.reader(open(os.path.join(OUT, "launches_bench.csv"))))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h, data = rows[hi], rows[hi + 1:]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    ours = [(r[ki], float(r[vi].replace(",", ""))) for r in data
            if len(r) > vi and r[mi] == "gpu__time_duration.sum" and r[ki].startswith(("void rl::", "rl::"))]
    with open(os.path.join(PROF, f"launches_{tag}.csv"), "w") as f:
        f.write("# ncu --metrics gpu__time_duration.sum --clock-control none, command: python bench.py "
                "--steps 2 --warmup 1 --no-e2e --no-cpu (cold-cache, serialised launches; compare shares)\n")
        f.write("# only this library's kernels (the step launches no others at N=1)\nkernel,ns\n")
        for k, v in ours:
            f.write(f"\"{k[:90]}\",{v:.0f}\n")
    agg = collections.defaultdict(list)
    for k, v in ours:
        agg[k.split("(")[0].replace("void ", "")[:70]].append(v)
    tot = sum(sum(v) for v in agg.values())
    lines = [f"{'kernel':72s} {'n':>5s} {'avg_us':>10s} {'share':>7s}"]
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"{k:72s} {len(v):5d} {sum(v) / len(v) / 1e3:10.1f} {100 * sum(v) / tot:6.2f}%")
    return "\n".join(lines)


UNITS = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    return dict(zip(r[0], r[2])), dict(zip(r[0], r[1]))


def main():
    tag = sys.argv[1]
    os.makedirs(PROF, exist_ok=True)
    summary = [f"# ncu evidence, round {tag}", "", "## Launch list of bench.py (our kernels)", "```",
               launches(tag), "```", ""]
    traffic = {}
    for name, rep, rows in (("sv", "prof_loss.ncu-rep", 16384), ("logprob", "prof_logprob.ncu-rep", 16384),
                            ("vp_finish", "prof_vpfin.ncu-rep", 16384)):
        p = os.path.join(OUT, rep)
        if not os.path.exists(p):
            continue
        d, units = raw(p)
        def g(k):
            try:
                return float(d[k].replace(",", ""))
            except (KeyError, ValueError):
                return float("nan")
        rd = g("dram__bytes_read.sum") * UNITS[units["dram__bytes_read.sum"]]
        wr = g("dram__bytes_write.sum") * UNITS[units["dram__bytes_write.sum"]]
        unit = 1.0
        per_tok = (rd + wr) / rows
        launch_rows = 65536 if name == "vp_finish" else 131072  # the bench's launch of that kernel
        traffic[name] = {"dram_bytes_per_launch": per_tok * launch_rows, "dram_bytes_per_token": per_tok,
                         "captured_rows": rows, "read_bytes": rd * unit, "write_bytes": wr * unit,
                         "note": f"ncu --set full of a {rows}-row launch; per-launch figure scaled to the "
                                 f"bench's {launch_rows}-row launch"}
        cols = 37984 if name == "vp_finish" else 151936
        summary += [f"## ncu --set full: {name} kernel ({rows} rows x {cols} bf16 columns)", "```"]
        for k in ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
                  "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
                  "sm__throughput.avg.pct_of_peak_sustained_elapsed",
                  "smsp__issue_active.avg.pct_of_peak_sustained_active",
                  "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
                  "lts__t_sector_hit_rate.pct", "launch__registers_per_thread", "launch__grid_size",
                  "launch__block_size", "launch__cluster_dim_x" if "launch__cluster_dim_x" in d else "launch__grid_size",
                  "sm__ctas_launched.sum"]:
            if k in d:
                summary.append(f"{k:60s} {d[k]} {units.get(k, '')}")
        alg = {"sv": 2 * 151936 * 2 + 17, "logprob": 151936 * 2 + 12, "vp_finish": 2 * 37984 * 2 + 17}[name]
        summary.append(f"{'algorithmic bytes per token':60s} {alg}")
        summary.append(f"{'dram bytes per token (measured)':60s} {per_tok:.0f}")
        st = sorted(((k, g(k)) for k in d if k.startswith("smsp__pcsamp_warps_issue_stalled")
                     and not k.endswith("not_issued")), key=lambda kv: -kv[1])
        tot = sum(v for _, v in st if v == v)
        summary.append("stall reasons (pc sampling):")
        for k, v in st[:8]:
            summary.append(f"   {k.replace('smsp__pcsamp_warps_issue_stalled_', ''):28s} {100 * v / tot:6.2f}%")
        summary += ["```", ""]
    with open(os.path.join(PROF, "ncu_traffic.json"), "w") as f:
        json.dump(traffic, f, indent=1)
    with open(os.path.join(PROF, f"ncu_summary_{tag}.md"), "w") as f:
        f.write("\n".join(summary) + "\n")
    print("\n".join(summary))


if __name__ == "__main__":
    main()
