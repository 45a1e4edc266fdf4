"""Summarise ncu --set full reports: duration, DRAM bytes, tensor / memory utilisation per kernel.
    python profiles/ncu_summary.py gpurun_out/prof_gemm6.ncu-rep [--json out.json]"""
import csv
import io
import json
import re
import subprocess
import sys

WANT = {
    "dur_us": "gpu__time_duration.sum",
    "dram_read": "dram__bytes_read.sum",
    "dram_write": "dram__bytes_write.sum",
    "dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "tensor_pct": "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "l2_pct": "lts__t_sectors.avg.pct_of_peak_sustained_elapsed",
    "regs": "launch__registers_per_thread",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "us": 1, "ms": 1e3, "ns": 1e-3, "msecond": 1e3,
         "usecond": 1, "nsecond": 1e-3}


def rows(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    h, units = r[0], r[1]
    res = []
    for row in r[2:]:
        d = {"kernel": re.sub(r"\(.*", "", row[h.index("Kernel Name")]).replace("void ", "").replace("unnamed>::", "")}
        for k, m in WANT.items():
            if m in h:
                i = h.index(m)
                try:
                    v = float(row[i].replace(",", ""))
                except ValueError:
                    continue
                d[k] = v * SCALE.get(units[i], 1)
        res.append(d)
    return res


if __name__ == "__main__":
    res = rows(sys.argv[1])
    for d in res:
        print(f"{d['kernel'][:45]:45s} {d.get('dur_us', 0):8.1f} us  DRAM r/w {d.get('dram_read', 0) / 1e6:7.1f}/"
              f"{d.get('dram_write', 0) / 1e6:6.1f} MB  dram% {d.get('dram_pct', 0):5.1f}  sm% {d.get('sm_pct', 0):5.1f}"
              f"  tensor% {d.get('tensor_pct', 0):5.1f}  regs {d.get('regs', 0):.0f}")
    if "--json" in sys.argv:
        json.dump(res, open(sys.argv[sys.argv.index("--json") + 1], "w"), indent=1)
