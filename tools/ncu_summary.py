"""Per-launch summary of an `ncu --set full` report, and the DRAM traffic per
kernel that bench.py reports as roofline.traffic.

  python tools/ncu_summary.py REPORT.ncu-rep OUT.csv [TRAFFIC.json]

OUT.csv: kernel, grid, duration, DRAM bytes read/written, achieved DRAM
GB/s, issue-slot and FP64-pipe utilisation, warps per SM, registers,
occupancy limits. TRAFFIC.json: {kernel name: mean DRAM bytes per launch}
(the kernel name as bench.py keys it, template arguments included)."""
import csv
import io
import json
import re
import subprocess
import sys

COLS = [
    ("duration_us", "gpu__time_duration.sum", 1e-3),  # ncu reports ns or us; normalised below
    ("dram_read_bytes", "dram__bytes_read.sum", 1.0),
    ("dram_write_bytes", "dram__bytes_write.sum", 1.0),
    ("issue_active_pct", "smsp__issue_active.avg.pct_of_peak_sustained_active", 1.0),
    ("fp64_pipe_pct", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", 1.0),
    ("warps_per_sm", "sm__warps_active.avg.per_cycle_active", 1.0),
    ("registers", "launch__registers_per_thread", 1.0),
    ("occ_limit_regs", "launch__occupancy_limit_registers", 1.0),
    ("occ_limit_smem", "launch__occupancy_limit_shared_mem", 1.0),
]
SCALE = {"ns": 1e-3, "us": 1.0, "ms": 1e3, "s": 1e6, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9,
         "KB": 1e3, "MB": 1e6, "GB": 1e9}


def short(name):
    name = re.sub(r"\([\w:]+\)$", "", name)  # drop the argument list
    name = name.replace("void ", "").replace("tmg::", "").replace("(bool)", "")
    return name


def main():
    rep, out = sys.argv[1], sys.argv[2]
    traffic_path = sys.argv[3] if len(sys.argv) > 3 else None
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units, data = rows[0], rows[1], rows[2:]
    ix = {h: k for k, h in enumerate(head)}
    res = []
    for r in data:
        d = {"kernel": short(r[ix["Kernel Name"]]), "grid": r[ix["Grid Size"]]}
        for key, metric, _ in COLS:
            v = float(r[ix[metric]].replace(",", ""))
            u = units[ix[metric]]
            if key == "duration_us":
                v *= SCALE.get(u, 1.0)
            elif key.startswith("dram"):
                v *= SCALE.get(u, 1.0)
            d[key] = v
        d["dram_gbs"] = (d["dram_read_bytes"] + d["dram_write_bytes"]) / (d["duration_us"] * 1e-6) / 1e9
        res.append(d)
    with open(out, "w", newline="") as fh:
        w = csv.DictWriter(fh, fieldnames=list(res[0].keys()))
        w.writeheader()
        for d in res:
            w.writerow({k: (f"{v:.4g}" if isinstance(v, float) else v) for k, v in d.items()})
    for d in res:
        print(f"{d['kernel'][:40]:40s} {d['grid']:>12s} {d['duration_us']:9.1f} us "
              f"{(d['dram_read_bytes'] + d['dram_write_bytes']) / 1e9:7.3f} GB {d['dram_gbs']:7.0f} GB/s "
              f"issue {d['issue_active_pct']:5.1f}% fp64 {d['fp64_pipe_pct']:5.1f}%")
    if traffic_path:
        acc = {}
        for d in res:
            acc.setdefault(d["kernel"], []).append(d["dram_read_bytes"] + d["dram_write_bytes"])
        # only the largest grid of a kernel name (the finest level it runs on)
        best = {}
        for d in res:
            k = d["kernel"]
            if k not in best or d["duration_us"] > best[k]["duration_us"]:
                best[k] = d
        json.dump({k: v["dram_read_bytes"] + v["dram_write_bytes"] for k, v in best.items()},
                  open(traffic_path, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
