"""Per-kernel roofline of one bench step from an ncu metrics capture (profiles/r01_roof_v10.csv):
duration, DRAM bytes, achieved DRAM bandwidth vs the measured HBM copy peak, tensor-pipe share, SM-active
share.  Usage: python profiles/roofline_table.py profiles/r01_roof_v10.csv [--per-step 20]"""
import csv
import json
import os
import re
import sys
from collections import OrderedDict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main(path, per_step=20):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, ii, mi, vi, ui = (h.index("Kernel Name"), h.index("ID"), h.index("Metric Name"), h.index("Metric Value"),
                          h.index("Metric Unit"))
    launches = OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        d = launches.setdefault(r[ii], {"kernel": re.sub(r"\(.*", "", r[ki]).replace("void ", "").replace("unnamed>::", "")
                                        .replace("luffy::", "").lstrip("<")})
        v = float(r[vi].replace(",", ""))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "ns": 1e-3, "usecond": 1,
                 "us": 1, "msecond": 1e3, "ms": 1e3}
        d[r[mi]] = v * scale.get(r[ui], 1)
    # one whole step of libluffy kernels: the last window that starts at the routing kernel (torch's own
    # kernels of the bench harness, e.g. the e2e result check, are not part of the step)
    mine = [d for d in launches.values() if not d["kernel"].startswith("at::")]
    starts = [i for i, d in enumerate(mine) if d["kernel"].lstrip("<").startswith("route_") and "bwd" not in d["kernel"]
              and i + per_step <= len(mine)]
    s0 = starts[-1] if starts else len(mine) - per_step
    last = mine[s0:s0 + per_step]
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs", 6547.5) \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6547.5
    tot = sum(d["gpu__time_duration.sum"] for d in last)
    out = ["| kernel | us (cold) | share | DRAM MB | GB/s | of HBM peak | tensor pipe | SM active |", "|---|---|---|---|---|---|---|---|"]
    for d in last:
        us = d["gpu__time_duration.sum"]
        mb = (d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)) / 1e6
        gbs = mb * 1e3 / us if us else 0
        act = d.get("sm__cycles_active.avg", 0) / max(1.0, d.get("sm__cycles_elapsed.avg", 1))
        out.append(f"| {d['kernel'][:48]} | {us:.1f} | {100 * us / tot:.1f} % | {mb:.1f} | {gbs:.0f} | "
                   f"{100 * gbs / peak:.0f} % | {d.get('sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed', 0):.0f} % | "
                   f"{100 * act:.0f} % |")
    out.append(f"| total ({len(last)} launches) | {tot:.1f} | | | | | | |")
    return "\n".join(out)


if __name__ == "__main__":
    n = int(sys.argv[sys.argv.index("--per-step") + 1]) if "--per-step" in sys.argv else 20
    print(main(sys.argv[1], n))
