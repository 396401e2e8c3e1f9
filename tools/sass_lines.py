"""Instructions executed per SOURCE line of one kernel: ncu's per-SASS
counts (source page of an `ncu --set full` report) joined by position with
`nvdisasm --print-line-info` of the same build.

  python tools/sass_lines.py REPORT.ncu-rep SKIP MANGLED_NAME [TOP]

Run against the library build the report was taken with."""
import collections
import csv
import io
import pathlib
import re
import subprocess
import sys
import tempfile

ROOT = pathlib.Path(__file__).resolve().parents[1]


def sass_lines(mangled):
    with tempfile.TemporaryDirectory() as d:
        subprocess.run(["cuobjdump", "-xelf", "all", str(ROOT / "paper_2301_07457_b200" / "libtmg_gpu.so")], cwd=d,
                       check=True, capture_output=True)
        cub = [p for p in pathlib.Path(d).glob("*.cubin") if "inputs" not in p.name][0]
        txt = subprocess.run(["nvdisasm", "--print-line-info", str(cub)], capture_output=True, text=True).stdout
    sec = txt[txt.index(f".text.{mangled}:"):]
    end = sec.find("//--------------------- .text.", 10)
    sec = sec[:end] if end > 0 else sec
    out, cur = [], ("?", 0)
    for ln in sec.split("\n"):
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m:
            cur = (pathlib.Path(m.group(1)).name, int(m.group(2)))
            continue
        if re.match(r"\s+/\*[0-9a-f]{4,}\*/", ln):
            out.append((cur, ln.split("*/", 1)[1].strip().split(";")[0]))
    return out


def main():
    rep, skip, mangled = sys.argv[1], int(sys.argv[2]), sys.argv[3]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
    res = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--launch-skip", str(skip), "--launch-count",
                          "1", "--print-source", "sass"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(res)))
    hdr = rows[1]
    data = []
    for r in rows[2:]:
        if len(r) > 5 and r[0].startswith("0x"):
            data.append(r)
        elif data:
            break
    ii = hdr.index("Instructions Executed")
    si = hdr.index("Warp Stall Sampling (All Samples)")
    sl = sass_lines(mangled)
    n = min(len(sl), len(data))
    mism = sum(1 for k in range(n) if sl[k][1].split()[0].lstrip("@!P0123456789U ") and
               sl[k][1].split()[-1:] != data[k][1].strip().split()[-1:])
    print(f"{len(sl)} SASS lines in build, {len(data)} in report, last-token mismatches {mism}")
    agg = collections.Counter()
    smp = collections.Counter()
    for k in range(n):
        agg[sl[k][0]] += float(data[k][ii] or 0)
        smp[sl[k][0]] += float(data[k][si] or 0)
    tot = sum(agg.values())
    ts = sum(smp.values())
    for (f, line), v in agg.most_common(top):
        print(f"{v / tot * 100:5.1f}% instr {smp[(f, line)] / ts * 100:5.1f}% samples  {f}:{line}")


if __name__ == "__main__":
    main()
