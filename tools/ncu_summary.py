"""Summarise an ncu --set full capture as markdown (key throughput, traffic,
occupancy and stall metrics, plus the opcode mix).  Not part of the product.

    python tools/ncu_summary.py REPORT.ncu-rep "title" [units_of_work] [unit_name]
        [--json WORKLOAD]   also merge the key counters into profiles/ncu_metrics.json
                            (read by bench.py's roofline.ncu)
"""
import json
import os
import collections
import csv
import io
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__registers_per_thread", "registers / thread"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active (% of peak)"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active (%)"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput (% of peak)"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1 throughput (% of peak)"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate (%)"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput (% of peak)"),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "threads per warp instruction"),
    ("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "global load sectors"),
    ("l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "global load requests"),
]


def _num(v):
    try:
        return float(str(v).replace(",", ""))
    except ValueError:
        return None


def ncu_csv(rep, *args):
    out = subprocess.run(["ncu", "-i", rep, *args, "--csv"], capture_output=True, text=True,
                         check=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main():
    argv = list(sys.argv[1:])
    workload = None
    if "--json" in argv:
        k = argv.index("--json")
        workload = argv[k + 1]
        del argv[k:k + 2]
    rep, title = argv[0], argv[1]
    units = float(argv[2]) if len(argv) > 2 else None
    uname = argv[3] if len(argv) > 3 else "unit"
    raw = ncu_csv(rep, "--page", "raw")
    hdr, unit_row, vals = raw[0], raw[1], raw[2]
    kname = vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
    print(f"# {title}\n")
    print(f"Kernel: `{kname}`  \nReport: `{rep}` (`ncu --set full --clock-control none`)\n")
    print("| metric | value |\n|---|---|")
    inst = None
    for m, label in METRICS:
        if m in hdr:
            v, u = vals[hdr.index(m)], unit_row[hdr.index(m)]
            print(f"| {label} (`{m}`) | {v} {u} |")
            if m == "smsp__inst_executed.sum":
                inst = float(v.replace(",", ""))
    if units and inst:
        print(f"| warp instructions per {uname} | {inst / units:.2f} |")
    # base units: bytes and nanoseconds (ncu scales each value's unit on its own)
    scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "s": 1e9, "ms": 1e6,
             "us": 1e3, "usecond": 1e3, "msecond": 1e6, "second": 1e9, "ns": 1.0, "nsecond": 1.0}

    def _base(m):
        v = _num(vals[hdr.index(m)])
        return None if v is None else v * scale.get(unit_row[hdr.index(m)].strip(), 1.0)

    get = {m: _base(m) for m, _ in METRICS if m in hdr}
    sec, req = (get.get("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum"),
                get.get("l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum"))
    tpi = get.get("smsp__thread_inst_executed_per_inst_executed.ratio")
    if sec and req:
        print(f"| global load sectors per request | {sec / req:.2f} |")
    if tpi:
        print(f"| warp execution efficiency (threads per instruction / 32) | {tpi / 32:.3f} |")
    if workload:
        path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                            "profiles", "ncu_metrics.json")
        try:
            with open(path) as f:
                allm = json.load(f)
        except Exception:
            allm = {}
        dram = (get.get("dram__bytes_read.sum") or 0) + (get.get("dram__bytes_write.sum") or 0)
        allm[workload] = {
            "kernel": kname, "report": os.path.basename(rep),
            "duration_ns": get.get("gpu__time_duration.sum"),
            "lts_throughput_pct": get.get("lts__throughput.avg.pct_of_peak_sustained_elapsed"),
            "dram_throughput_pct": get.get("dram__throughput.avg.pct_of_peak_sustained_elapsed"),
            "l2_hit_rate_pct": get.get("lts__t_sector_hit_rate.pct"),
            "l1tex_throughput_pct": get.get("l1tex__throughput.avg.pct_of_peak_sustained_active"),
            "issue_active_pct": get.get("smsp__issue_active.avg.pct_of_peak_sustained_active"),
            "warps_active_pct": get.get("sm__warps_active.avg.pct_of_peak_sustained_active"),
            "sectors_per_request": (sec / req) if (sec and req) else None,
            "warp_execution_efficiency": (tpi / 32) if tpi else None,
            "dram_bytes": dram or None,
            "warp_instructions": inst,
            "warp_instructions_per_unit": (inst / units) if (units and inst) else None,
            "unit": uname if units else None,
        }
        with open(path, "w") as f:
            json.dump(allm, f, indent=1)
    stalls = []
    for i, h in enumerate(hdr):
        if "issue_stalled" in h and h.endswith("per_issue_active.ratio"):
            try:
                stalls.append((float(vals[i]), h))
            except ValueError:
                pass
    print("\nTop stall reasons (warps stalled per issued instruction):\n")
    for v, h in sorted(stalls, reverse=True)[:6]:
        name = h.replace("smsp__average_warps_issue_stalled_", "").replace(
            "_per_issue_active.ratio", "")
        print(f"- {name}: {v:.2f}")
    src = ncu_csv(rep, "--page", "source", "--print-source", "sass")
    shdr = src[1]
    si, ei = shdr.index("Source"), shdr.index("Instructions Executed")
    ops = collections.Counter()
    tot = 0
    for r in src[2:]:
        try:
            e = int(r[ei])
        except (ValueError, IndexError):
            continue
        t = r[si].strip().split()
        if not t:
            continue
        op = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
        ops[op] += e
        tot += e
    print("\nOpcode mix (share of executed warp instructions):\n")
    print(", ".join(f"{o} {100 * e / tot:.1f} %" for o, e in ops.most_common(12)))


if __name__ == "__main__":
    main()
