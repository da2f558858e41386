"""Turns the ncu outputs of a round into the committed summaries.

    python profiles/summarize.py <round> <launches.csv> [<full.ncu-rep>]

Writes profiles/<round>_launches.csv (copy), profiles/<round>_summary.md and
merges per-launch DRAM traffic of the top kernels into profiles/traffic.json
(read by bench.py for the roofline's `traffic` field)."""
import csv
import json
import os
import shutil
import subprocess
import sys
from collections import defaultdict

HERE = os.path.dirname(os.path.abspath(__file__))


def short(name):
    for k in ("tbe_forward", "sgd_seg_kernel", "sgd_carry_kernel", "sgd_kernel", "sort_count",
              "sort_scan", "sort_scatter", "sort_bucket", "sort_big", "narrow_table",
              "rollout", "eval_kernel"):
        if k in name:
            return k
    return name[:40]


def launches(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    n, mn, v = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    per = defaultdict(dict)
    names = {}
    for r in rows[start + 1:]:
        per[int(r[0])][r[mn]] = float(r[v].replace(",", ""))
        names[int(r[0])] = short(r[n])
    return [(i, names[i], per[i]) for i in sorted(per)]


def full_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[0]
    want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum",
            "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
            "sm__warps_active.avg.per_cycle_active", "launch__registers_per_thread",
            "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
            "lts__throughput.avg.pct_of_peak_sustained_elapsed"]
    res = []
    for r in rows[2:]:
        d = {}
        for w in want:
            if w in hdr:
                d[w] = r[hdr.index(w)]
        d["units"] = {w: rows[1][hdr.index(w)] for w in want if w in hdr}
        res.append(d)
    return res


def to_bytes(val, unit):
    f = float(val.replace(",", ""))
    return f * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)


def main():
    rnd, lpath = sys.argv[1], sys.argv[2]
    rep = sys.argv[3] if len(sys.argv) > 3 else None
    # the commit the capture ran (gpurun snapshots the committed tree)
    head = subprocess.run(["git", "rev-parse", "--short=12", "HEAD"], capture_output=True,
                          text=True, cwd=HERE).stdout.strip()
    shutil.copy(lpath, os.path.join(HERE, f"{rnd}_launches.csv"))
    L = launches(lpath)
    lines = [f"# {rnd}: ncu summary (cfg3, D=1, one iteration = the launches below)", "",
             "Launch list (`--metrics gpu__time_duration.sum,dram__bytes_*` "
             "`--clock-control none`, cold-cache and serialised: compare shares):", "",
             "| id | kernel | µs | DRAM read MB | DRAM write MB |", "|---|---|---|---|---|"]
    for i, name, m in L:
        lines.append(f"| {i} | {name} | {m.get('gpu__time_duration.sum', 0) / 1e3:.1f} | "
                     f"{m.get('dram__bytes_read.sum', 0) / 1e6:.0f} | "
                     f"{m.get('dram__bytes_write.sum', 0) / 1e6:.0f} |")
    traffic_path = os.path.join(HERE, "traffic.json")
    traffic = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
    if rep:
        lines += ["", f"Full capture (`ncu --set full`, `{os.path.basename(rep)}`):", "",
                  "| kernel | ms | DRAM read | DRAM write | L2 hit % | warps/SM | regs | "
                  "long-scoreboard stall | LTS % |", "|---|---|---|---|---|---|---|---|---|"]
        for d in full_metrics(rep):
            u = d["units"]
            lines.append("| " + " | ".join([
                short(d.get("Kernel Name", "")), d.get("gpu__time_duration.sum", ""),
                d.get("dram__bytes_read.sum", "") + " " + u.get("dram__bytes_read.sum", ""),
                d.get("dram__bytes_write.sum", "") + " " + u.get("dram__bytes_write.sum", ""),
                d.get("lts__t_sector_hit_rate.pct", ""),
                d.get("sm__warps_active.avg.per_cycle_active", ""),
                d.get("launch__registers_per_thread", ""),
                d.get("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", ""),
                d.get("lts__throughput.avg.pct_of_peak_sustained_elapsed", "")]) + " |")
            k = {"tbe_forward": "fwd", "sgd_kernel": "sgd", "sgd_seg_kernel": "sgd",
                 "sort_scatter": "sort_scatter", "sort_big": "sort_big"}.get(
                     short(d.get("Kernel Name", "")))
            if k:
                traffic[f"cfg3/D1/{k}"] = {
                    "dram_bytes": to_bytes(d["dram__bytes_read.sum"], u["dram__bytes_read.sum"]) +
                    to_bytes(d["dram__bytes_write.sum"], u["dram__bytes_write.sum"]),
                    "head": head, "capture": os.path.basename(rep)}
        json.dump(traffic, open(traffic_path, "w"), indent=1)
    open(os.path.join(HERE, f"{rnd}_summary.md"), "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
