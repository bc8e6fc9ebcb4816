"""Summarise ncu evidence into profiles/: per-kernel share of a launch list
(gpu__time_duration, cold-cache serialised) and the key counters of
`--set full` captures (DRAM bytes, throughput, occupancy, stalls).

    python tools/ncu_summary.py <round> <launches.csv> <capture.ncu-rep>...
"""

from __future__ import annotations

import collections
import csv
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio"]


def launches(path: Path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in rows[hi + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki].split("(")[0].split("<")[0].replace("void ", "").replace("gdsw::", "")
        tot[name] += float(r[vi].replace(",", ""))
        cnt[name] += 1
    total = sum(tot.values())
    return [dict(kernel=k, launches=cnt[k], total_us=v / 1e3, avg_us=v / cnt[k] / 1e3,
                 share=v / total) for k, v in sorted(tot.items(), key=lambda x: -x[1])]


def capture(path: Path):
    out = subprocess.run(["ncu", "-i", str(path), "--page", "raw", "--csv"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, u, v = rows[0], rows[1], rows[2]
    name = v[h.index("Kernel Name")].split("(")[0].split("<")[0].replace("void ", "")
    d = {"kernel": name.replace("gdsw::", ""), "capture": path.name}
    for k in KEYS:
        if k in h:
            i = h.index(k)
            try:
                d[k] = float(v[i].replace(",", ""))
            except ValueError:
                d[k] = v[i]
            d[k + ".unit"] = u[i]
    rd, wr = d.get("dram__bytes_read.sum"), d.get("dram__bytes_write.sum")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    if rd is not None:
        d["traffic_bytes"] = (rd * scale[d["dram__bytes_read.sum.unit"]]
                              + wr * scale[d["dram__bytes_write.sum.unit"]])
    return d


def main():
    rnd, lst, caps = sys.argv[1], Path(sys.argv[2]), [Path(p) for p in sys.argv[3:]]
    L = launches(lst)
    C = [capture(p) for p in caps]
    prof = ROOT / "profiles"
    prof.mkdir(exist_ok=True)
    (prof / f"{rnd}_ncu_summary.json").write_text(json.dumps({"launches": L, "captures": C},
                                                             indent=1))
    lines = [f"# ncu summary {rnd}", "",
             f"Launch list `{lst.name}` (ncu --metrics gpu__time_duration.sum --clock-control none,"
             " one C2 solve, cold-cache serialised launches: compare shares, not absolutes).", "",
             "| kernel | launches | total us | avg us | share |", "|---|---|---|---|---|"]
    for r in L:
        lines.append(f"| {r['kernel']} | {r['launches']} | {r['total_us']:.0f} | {r['avg_us']:.1f} |"
                     f" {100 * r['share']:.1f}% |")
    lines += ["", "`--set full` captures (one launch each):", "",
              "| kernel | us | DRAM read+write MB | DRAM % peak | L2 hit % | warps active % | regs |"
              " long-scoreboard stall/issue |", "|---|---|---|---|---|---|---|---|"]
    for c in C:
        lines.append(
            f"| {c['kernel']} | {c.get('gpu__time_duration.sum', '')} | "
            f"{c.get('traffic_bytes', 0) / 1e6:.1f} | "
            f"{c.get('gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', '')} | "
            f"{c.get('lts__t_sector_hit_rate.pct', '')} | "
            f"{c.get('sm__warps_active.avg.pct_of_peak_sustained_active', '')} | "
            f"{c.get('launch__registers_per_thread', '')} | "
            f"{c.get('smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio', '')} |")
    (prof / f"{rnd}_ncu_summary.md").write_text("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
