"""Map ncu SASS-level stall samples of one kernel to CUDA source lines (needs -lineinfo).
    python tools/ncu_lines.py REPORT.ncu-rep KERNEL_MANGLED_NAME [--top 30]"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    rep, kern = sys.argv[1], sys.argv[2]
    top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 30
    lib = os.path.join(ROOT, "paper_2605_15565_b200", "librlpolicy.so")
    with tempfile.TemporaryDirectory() as td:
        subprocess.run(["cuobjdump", "-xelf", "all", lib], cwd=td, capture_output=True)
        dis = ""
        for f in os.listdir(td):
            if f.endswith(".cubin"):
                out = subprocess.run(["nvdisasm", "-g", os.path.join(td, f)], capture_output=True, text=True).stdout
                if f".text.{kern}:" in out:
                    dis = out
                    break
    lines = dis.split("\n")
    start = [i for i, l in enumerate(lines) if l.startswith(f".text.{kern}:")][0]
    cur, off2line = None, {}
    for ln in lines[start + 1:]:
        if ln.startswith(".text.") or ln.startswith(".nv."):
            break
        m = re.search(r'//## File "(.*?)", line (\d+)', ln)
        if m:
            cur = (m.group(1).split("/")[-1], int(m.group(2)))
            continue
        m = re.search(r"/\*([0-9a-f]{4,})\*/", ln)
        if m and cur is not None:
            off2line[int(m.group(1), 16)] = cur
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, data = rows[1], rows[2:]
    ia, ist, ie = h.index("Address"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
    base = int(data[0][ia], 16)
    by, inst = collections.Counter(), collections.Counter()
    for r in data:
        l = off2line.get(int(r[ia], 16) - base, ("?", -1))
        by[l] += int(r[ist] or 0)
        inst[l] += int(r[ie] or 0)
    tot = sum(by.values())
    srcs = {}
    for d, _, fs in os.walk(os.path.join(ROOT, "paper_2605_15565_b200", "csrc")):
        for f in fs:
            srcs[f] = open(os.path.join(d, f)).read().split("\n")
    for l, c in by.most_common(top):
        txt = srcs[l[0]][l[1] - 1].strip()[:80] if l[0] in srcs and l[1] > 0 else ""
        print(f"{100 * c / tot:5.1f}% {l[0]:>24}:{l[1]:<4} inst {inst[l]:>10}  {txt}")


if __name__ == "__main__":
    main()
