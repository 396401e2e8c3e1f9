"""Instruction mix and stall samples per opcode from an ncu report's SASS
source page:  python tools/sass_mix.py REPORT.ncu-rep [kernel-substring] [top]

Reads `ncu -i REPORT --page source --csv --print-source sass` (every profiled
kernel, one section each) and prints, per kernel, warp instructions executed
and warp-stall samples grouped by opcode (modifiers stripped)."""
import collections
import csv
import io
import subprocess
import sys


def sections(report):
    out = subprocess.run(["ncu", "-i", report, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True, check=True).stdout
    cur, name = [], None
    for line in out.splitlines():
        if line.startswith('"Kernel Name"'):
            if name:
                yield name, cur
            name, cur = next(csv.reader(io.StringIO(line)))[1], []
        else:
            cur.append(line)
    if name:
        yield name, cur


def main():
    report = sys.argv[1]
    want = sys.argv[2] if len(sys.argv) > 2 else ""
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
    seen = set()
    for name, lines in sections(report):
        if want not in name or name in seen:
            continue
        seen.add(name)
        rows = list(csv.DictReader(io.StringIO("\n".join(lines))))
        ins = collections.Counter()
        stall = collections.Counter()
        for r in rows:
            src = r.get("Source", "").strip()
            if not src:
                continue
            op = src.split()[0]
            if op.startswith("@"):
                op = src.split()[1]
            op = op.split(".")[0]
            ins[op] += float(r.get("Instructions Executed") or 0)
            stall[op] += float(r.get("Warp Stall Sampling (All Samples)") or 0)
        ti, ts = sum(ins.values()) or 1, sum(stall.values()) or 1
        print(f"== {name}: {ti:.4g} warp instructions, {ts:.0f} stall samples")
        for op, n in ins.most_common(top):
            print(f"  {op:12s} {n / ti * 100:6.2f}% inst   {stall[op] / ts * 100:6.2f}% samples")


if __name__ == "__main__":
    main()
