"""Summarise an ncu --set full report: headline metrics, stall reasons, opcode mix, top lines.
    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [--top 20]"""
import collections
import csv
import io
import subprocess
import sys


def ncu_csv(rep, *args):
    out = subprocess.run(["ncu", "-i", rep, *args, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main():
    rep = sys.argv[1]
    top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 20
    r = ncu_csv(rep, "--page", "raw")
    h, v = r[0], r[2]
    d = dict(zip(h, v))

    def f(k):
        try:
            return float(d.get(k, "nan").replace(",", ""))
        except ValueError:
            return float("nan")
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
            "lts__t_sector_hit_rate.pct", "smsp__inst_executed.sum", "launch__registers_per_thread",
            "sm__warps_active.avg.pct_of_peak_sustained_active"]
    for k in keys:
        print(f"{k:60s} {d.get(k, '-')}")
    st = [(k, f(k)) for k in h if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued")]
    tot = sum(x for _, x in st if x == x)
    print("-- stall reasons (pc sampling)")
    for k, x in sorted(st, key=lambda kv: -kv[1])[:10]:
        print(f"   {k.replace('smsp__pcsamp_warps_issue_stalled_', ''):28s} {100 * x / tot:6.2f}%")
    s = ncu_csv(rep, "--page", "source", "--print-source", "sass")
    hh = s[1]
    data = s[2:]
    ia, ie, ist = hh.index("Source"), hh.index("Instructions Executed"), hh.index("Warp Stall Sampling (All Samples)")
    te = sum(int(x[ie] or 0) for x in data)
    ts = sum(int(x[ist] or 0) for x in data)
    op, ops = collections.Counter(), collections.Counter()
    for x in data:
        toks = x[ia].strip().split()
        if not toks:
            continue
        o = toks[1] if toks[0].startswith("@") else toks[0]
        o = o.split(".")[0]
        op[o] += int(x[ie] or 0)
        ops[o] += int(x[ist] or 0)
    print(f"-- opcode mix (executed warp instructions: {te})")
    for o, c in op.most_common(top):
        print(f"   {o:12s} {100 * c / te:6.2f}% inst  {100 * ops[o] / max(ts, 1):6.2f}% stall samples")
    print("-- top SASS lines by stall samples")
    for x in sorted(data, key=lambda x: -int(x[ist] or 0))[:top]:
        print(f"   {x[ist]:>7s} {x[ie]:>10s}  {x[ia].strip()[:80]}")


if __name__ == "__main__":
    main()
