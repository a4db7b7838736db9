"""Summarise a run_once log (label line + dict line per run).  Not part of the product."""
import ast
import sys

lines = open(sys.argv[1]).read().splitlines()
for i, l in enumerate(lines):
    if l.startswith("cfg"):
        try:
            d = ast.literal_eval(lines[i + 1])
            print(l, {k: round(d[k], 2) for k in ("ms_total", "ms_sample", "ms_gather", "ms_extras")},
                  d["edges"], round(d["gather_bytes"] / d["gather_pairs"], 2), d.get("filter_bits"))
        except Exception:
            print(l, lines[i + 1][:300] if i + 1 < len(lines) else "")
