"""Markdown table of committed bench lines (profiles/r02_bench/*.json): one row per JSON line.
    python tools/status_table.py profiles/r02_bench/*.json"""
import json
import sys


def last_json(path):
    with open(path) as fh:
        lines = [ln for ln in fh.read().strip().splitlines() if ln.startswith("{")]
    return json.loads(lines[-1]) if lines else None


print("| file | N | workload | h | tokens/s | ms/step | e2e tokens/s | roofline (bound, frac) | Gram frac | memory frac | condensed | SM MHz |")
print("|---|---|---|---|---|---|---|---|---|---|---|---|")
for p in sys.argv[1:]:
    d = last_json(p)
    if not d or "value" not in d:
        continue
    c = d.get("config", {})
    r = d.get("roofline") or {}
    g = d.get("roofline_gram") or {}
    m = d.get("roofline_memory") or {}
    e = d.get("e2e") or {}
    clk = (d.get("clocks") or {}).get("sm_mhz")
    cond = d.get("condensed_frac_rows")
    print(f"| {p.split('/')[-1]} | {d.get('n_gpus')} | {c.get('workload')} | {c.get('h', '')} | "
          f"{d['value'] / 1e6:.3f} M | {d['ms_per_step']:.3f} | "
          f"{(e.get('value') or 0) / 1e6:.3f} M | {r.get('bound', '')} {r.get('frac', 0):.2f} | "
          f"{g.get('frac', 0):.2f} | {m.get('frac', 0):.2f} | "
          f"{'' if cond is None else f'{cond:.2f}'} | {clk} |")
