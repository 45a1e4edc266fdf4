"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: the kernels of the last
`--per-step` launches (one bench step) with their share of the step.  Usage:
    python profiles/launch_summary.py gpurun_out/launches.csv [--per-step 21]"""
import csv
import re
import sys


def main(path, per_step=21):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, mi = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
    seq = [(r[ki], float(r[vi].replace(",", ""))) for r in rows[hi + 1:] if len(r) > vi and r[mi] == "gpu__time_duration.sum"]
    last = seq[-per_step:]
    tot = sum(v for _, v in last)
    out = []
    for n, v in last:
        short = re.sub(r"\(.*", "", n).replace("void ", "").replace("unnamed>::", "")
        out.append(f"{v / 1000:9.1f} us {100 * v / tot:5.1f}%  {short[:100]}")
    out.append(f"{tot / 1000:9.1f} us total over {len(last)} launches (cold-cache, serialised)")
    return "\n".join(out)


if __name__ == "__main__":
    n = int(sys.argv[sys.argv.index("--per-step") + 1]) if "--per-step" in sys.argv else 21
    print(main(sys.argv[1], n))
