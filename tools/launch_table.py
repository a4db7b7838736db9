"""Markdown table of an ncu launch list (--metrics gpu__time_duration.sum --csv):
kernels grouped by name, time per step and share.  Not part of the product.

    python tools/launch_table.py launches.csv STEPS "title" > profiles/<round>_launches.md
"""
import collections
import csv
import sys


def main(path, steps, title):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, vi, mi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
    t, c = collections.Counter(), collections.Counter()
    for r in rows[1:]:
        if r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki].replace("void ", "").replace("sngb::", "").replace("<unnamed>::", "")
        name = name.replace("unnamed>::", "").split("(")[0][:72]
        t[name] += float(r[vi].replace(",", "")) / 1e6  # ns -> ms
        c[name] += 1
    total = sum(t.values())
    print(f"# {title}\n")
    print("`ncu --metrics gpu__time_duration.sum --clock-control none` (cold caches, serialised "
          f"launches: the *share* is what matters).  {steps} steps captured; per-step = total / {steps}.\n")
    print("| kernel | launches | per step ms | share |\n|---|---|---|---|")
    for name, ms in t.most_common():
        print(f"| `{name}` | {c[name]} | {ms / steps:.3f} | {100 * ms / total:.1f} % |")
    print(f"\nTotal per step: {total / steps:.3f} ms")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]), sys.argv[3])
