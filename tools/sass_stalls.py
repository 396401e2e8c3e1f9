"""Per-instruction stall attribution of one kernel launch from an
`ncu --set full --import-source on` report (source page, SASS view).

  python tools/sass_stalls.py REPORT.ncu-rep [--skip K] [--reason long_sb] [--top 25]

Prints the stall-reason totals, then the instructions with the most samples
for the chosen reason (default: all samples), each with its source line."""
import argparse
import csv
import io
import subprocess


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--skip", type=int, default=0)
    ap.add_argument("--kernel", default=None)
    ap.add_argument("--reason", default=None)
    ap.add_argument("--top", type=int, default=25)
    a = ap.parse_args()
    cmd = ["ncu", "-i", a.report, "--page", "source", "--csv", "--launch-skip", str(a.skip), "--launch-count", "1",
           "--print-source", "sass"]
    if a.kernel:
        cmd += ["--kernel-name", f"regex:{a.kernel}"]
    out = subprocess.run(cmd, capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    print(" ".join(rows[0][:2]))
    hdr = rows[1]
    data = []
    for r in rows[2:]:
        if len(r) > 5 and r[0].startswith("0x"):
            data.append(r)
        elif data:
            break  # first launch only
    reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    tot = {h: sum(float(r[hdr.index(h)] or 0) for r in data) for h in reasons}
    allv = sum(tot.values()) or 1
    print("  ".join(f"{k[6:]} {v / allv * 100:.0f}%" for k, v in sorted(tot.items(), key=lambda kv: -kv[1]) if v))
    key = hdr.index("stall_" + a.reason) if a.reason else hdr.index("Warp Stall Sampling (All Samples)")
    order = sorted(range(len(data)), key=lambda i: -float(data[i][key] or 0))
    for i in order[: a.top]:
        r = data[i]
        print(f"{i:5d} {float(r[key] or 0):7.0f}  {r[1].strip()[:70]}")


if __name__ == "__main__":
    main()
