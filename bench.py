#!/usr/bin/env python
"""bench.py -- SNG-DBSCAN hot path on B200 (sampled pairs/s, e2e, roofline).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 1..5] [--impl reference]
    torchrun --nproc-per-node N bench.py --gpus N ...     (rows sharded over N GPUs)

With --gpus N > 1 and no torchrun environment, bench.py re-launches itself as
N ranks (python -m torch.distributed.run --nproc-per-node N ...), one per GPU.
The default workload is BASELINE.json's largest config that fits one GPU:
cfg5 (n = 20 M, d = 32); --config 1..4 selects the other shapes.

A "step" is one full sng::sng_dbscan (clusterer.cpp:54-65) over one synthetic
workload: sample + eps-test every vertex's draws, symmetrise/dedup, degrees,
core mask, union-find, border, relabel.  The metric is BASELINE.json's:
sampled pairs per second (pairs = n * draws, the reference's distance_evals),
end-to-end clustering time, and the gather kernel's fraction of roofline.

  value     device-resident: points already in HBM, labels left in HBM;
            CUDA events per step on the launching stream, L2 flushed (256 MB
            write) before every timed step, max over ranks.
  e2e       the public host API (sngb_dbscan_f32 through the C ABI) from
            pinned host memory: H2D of the points and D2H of labels+roles
            inside the timed region; its labels must equal the device-resident
            run's (checked every run).  e2e_pageable: the same call from the
            pageable numpy array the Python / C++ mirrors pass.
  roofline  the dominant kernel's own algorithmic bytes over its CUDA-event
            duration (measured inside the library on its stream) against the
            measured random-gather ceiling of the memory level it reads
            (tools/gather_ceiling.cu); frac_8d is SURVEY 8(d)'s 4*d bytes per
            pair against MEASURED_PEAKS.json hbm_gbs -- an effective rate (the
            filters read far fewer bytes), not a roofline fraction.
  cpu_baseline  the reference's own graph.cpp/clusterer.cpp (oracle/_ref,
            compiled unmodified) on this host's cores, rank 0, N=1 only, on the
            FULL dataset with fewer draws per vertex (a bounded sample).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "sampled_pairs_per_sec"
UNIT = "pairs/s"
DEFAULT_CONFIG = 5  # BASELINE.json configs[4]: the largest config that fits one GPU


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--config", type=int, default=DEFAULT_CONFIG, choices=[1, 2, 3, 4, 5])
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-pageable", action="store_true")
    p.add_argument("--cpu-budget-s", type=float, default=25.0,
                   help="CPU seconds allowed for the cpu_baseline sample")
    return p.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


Q8_SPLIT_MIN_RW, Q8_HEAD_BYTES, Q8_HEAD_VALS = 40, 256, 240  # sngb_internal.cuh kSplitMinRW, kHead


def load_gather_ceiling(d: int, n: int, row: int | None = None, read: int | None = None):
    """Measured random-row gather ceiling for this row shape and table size
    (tools/gather_ceiling.cu -> profiles/r01_gather_ceilings.jsonl): the best
    rows/s of a lean gather with no per-pair work, swept over rows in flight
    and blocks per SM.  Returns (case name, rows/s) or (None, None)."""
    path = os.path.join(ROOT, "profiles", "r01_gather_ceilings.jsonl")
    try:
        cases = [json.loads(ln) for ln in open(path) if ln.strip().startswith("{")]
    except Exception:
        return None, None
    if row is None:
        row = 8 if d <= 2 else 16 * ((d + 3) // 4)  # padded device row, bytes
    table = n * row
    # same row size; among those, the table size closest to ours (L2 vs HBM)
    same = [c for c in cases if c["row_bytes"] == max(row, 16)
            and c.get("read_bytes", c["row_bytes"]) == (read or c["row_bytes"])]
    if not same:
        return None, None
    best = min(same, key=lambda c: abs(math.log(c["table_MB"] * 2**20 / max(table, 1))))
    return best["bench"], best["rows_per_s"]


def load_head_ceiling(n: int, hb: int = 4):
    """Measured random hb-byte-row gather (the head table, n x hb bytes) closest in
    table size: (case name, rows/s) or (None, None)."""
    path = os.path.join(ROOT, "profiles", "r01_gather_ceilings.jsonl")
    try:
        cases = [json.loads(ln) for ln in open(path) if ln.strip().startswith("{")]
    except Exception:
        return None, None
    same = [c for c in cases if c["bench"].startswith(f"ceiling_head{hb}B")]
    if not same:
        return None, None
    best = min(same, key=lambda c: abs(math.log(c["table_MB"] * 2**20 / max(hb * n, 1))))
    return best["bench"], best["rows_per_s"]


def load_ncu(workload: str):
    """Key counters of the dominant kernel from the committed ncu --set full capture
    (profiles/ncu_metrics.json, written by tools/ncu_summary.py --json)."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_metrics.json")) as f:
            return json.load(f).get(workload)
    except Exception:
        return None


def load_traffic(workload: str):
    """dram bytes per gather launch from the committed ncu --set full capture."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            return json.load(f).get(workload)
    except Exception:
        return None


class ClockSampler:
    """SM clock + throttle reasons sampled during the timed region.

    NVML in-process (a 10 Hz thread; the GIL is released while the library call
    runs): an `nvidia-smi -lms 100` child cost the large configs ~5 ms of GPU
    stall per poll on some boxes (cfg4: an 88.0 ms step around an 82.9 ms call).
    Falls back to that child process when NVML is not importable."""

    Q = ("timestamp,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    NVML_REASONS = ((0x8, "hw_slowdown"), (0x40, "hw_thermal_slowdown"),
                    (0x20, "sw_thermal_slowdown"), (0x4, "sw_power_cap"))

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []
        self.samples = []  # (sm_mhz, reasons bitmask) from NVML
        self.mx = None
        self.thread = None
        self._stop = None
        self.source = None

    def _nvml_loop(self, nv, h):
        while not self._stop.is_set():
            try:
                self.samples.append((float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)),
                                     int(nv.nvmlDeviceGetCurrentClocksThrottleReasons(h))))
            except Exception:
                pass
            self._stop.wait(0.1)

    def start(self):
        if os.environ.get("SNGB_BENCH_CLOCKS") != "smi":
            try:
                import threading

                import pynvml as nv
                nv.nvmlInit()
                # NVML enumerates every GPU of the box: map the CUDA ordinal through its UUID
                import torch
                uuid = str(torch.cuda.get_device_properties(self.index).uuid)
                h = None
                for i in range(nv.nvmlDeviceGetCount()):
                    hi = nv.nvmlDeviceGetHandleByIndex(i)
                    u = nv.nvmlDeviceGetUUID(hi)
                    u = u.decode() if isinstance(u, bytes) else u
                    if uuid in u:
                        h = hi
                        break
                if h is None:
                    h = nv.nvmlDeviceGetHandleByIndex(self.index)
                self.mx = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
                self._stop = threading.Event()
                self.thread = threading.Thread(target=self._nvml_loop, args=(nv, h), daemon=True)
                self.thread.start()
                self.source = "nvml"
                return
            except Exception:
                self.thread = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100", "-i", str(self.index)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.source = "nvidia-smi -lms 100"
        except Exception:
            self.proc = None

    def stop(self):
        if self.thread:
            self._stop.set()
            self.thread.join(timeout=2)
            return
        if not self.proc:
            return
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out = ""
        self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def summary(self):
        if self.thread:
            sms = [a for a, _ in self.samples]
            bits = 0
            for _, r in self.samples:
                bits |= r
            return {"sm_mhz": statistics.median(sms) if sms else None, "sm_max_mhz": self.mx,
                    "reasons": sorted(nm for b, nm in self.NVML_REASONS if bits & b),
                    "samples": len(sms), "source": self.source}
        sms, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 8:
                continue
            try:
                sm = float(f[1])
                mx = float(f[2])
            except ValueError:
                continue
            sms.append(sm)
            for nm, v in zip(names, f[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sms) if sms else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sms), "source": self.source}


def _workload_config(w, n_gpus: int, extra: dict | None = None) -> dict:
    """The config dict both arms print (same keys, so the driver can match them)."""
    c = {"workload": w.name, "n": w.n, "d": w.d, "eps": w.eps, "rate": w.rate,
         "min_pts": w.min_pts, "seed": w.seed, "draws": w.draws, "pairs": w.pairs,
         "parallelism": f"rows sharded x{n_gpus}" if n_gpus > 1 else "1 GPU",
         "l2": "256 MB L2 flush before every timed step"}
    if extra:
        c.update(extra)
    return c


def _ref_rate(w, draws_s: int) -> float:
    """A rate whose draws = min(ceil(rate*n), n-1) is exactly draws_s (graph.cpp:139-140)."""
    n = w.n
    rate = draws_s / n
    while min(math.ceil(rate * float(n)), n - 1) > draws_s:
        rate = math.nextafter(rate, 0.0)
    while min(math.ceil(rate * float(n)), n - 1) < draws_s:
        rate = math.nextafter(rate, 1.0)
    return rate


def _ref_calibrate(ref, ds, w, budget_s: float) -> int:
    """Draws per vertex so one reference call on the full dataset takes at most
    ~0.8 budget_s: a tiny call (d0 draws), then one of about a quarter of the
    budget (d1, grown 4x at a time until it takes >= budget/8), and the line
    through the last two (fixed per-call cost + cost per draw).  The points
    are far apart, so a noisy fixed cost cannot skew the slope (a 1-vs-5-draw
    probe once mistook noise for throughput and ran the full workload)."""
    def timed(dr):
        t = ref.sng_dbscan(ds, w.eps, w.min_pts, _ref_rate(w, dr), w.seed, threads=0)[2]["ms"] / 1e3
        print(f"bench.py: reference calibration draws={dr} {t:.3f} s", file=sys.stderr)
        return t

    d0 = int(min(w.draws, max(1, (1e8 * 16 / max(w.d, 16)) // w.n)))
    t0 = timed(d0)
    # grow the second point until its draw work clearly dominates the fixed cost
    d1, t1 = d0, t0
    while t1 < 0.125 * budget_s and d1 < w.draws:
        d0, t0 = d1, t1
        d1 = int(min(w.draws, d1 * 4))
        t1 = timed(d1)
    if d1 <= d0 or t1 <= t0:  # no measurable per-draw cost: stay at the measured point
        return d1
    slope = (t1 - t0) / (d1 - d0)
    fixed = max(0.0, t0 - slope * d0)
    return int(max(1, min(w.draws, (0.8 * budget_s - fixed) / slope)))


def _sample_desc(w, draws_s: int) -> str:
    if draws_s >= w.draws:
        return f"full workload (n={w.n}, draws={w.draws})"
    return (f"the full dataset (n={w.n}, d={w.d}, same eps/min_pts/seed) with "
            f"draws={draws_s} per vertex instead of {w.draws} (rate={_ref_rate(w, draws_s):.6g}): "
            f"every pair still gathers a random partner row from the whole table")


def cpu_baseline(pts, w, budget_s: float):
    """The reference's own sng_dbscan (oracle/_ref) on all host cores, on the full
    dataset, with as many draws per vertex as fit `budget_s`."""
    from oracle import Reference
    ref = Reference()
    cores = ref.hw_threads()
    ds = ref.dataset(pts)
    draws_s = _ref_calibrate(ref, ds, w, budget_s)
    rate = w.rate if draws_s >= w.draws else _ref_rate(w, draws_s)
    _, _, info = ref.sng_dbscan(ds, w.eps, w.min_pts, rate, w.seed, threads=0)
    pairs = info["distance_evals"]
    return {"value": pairs / (info["ms"] / 1e3), "unit": UNIT, "cores": cores,
            "kind": "reference", "sample": _sample_desc(w, draws_s), "ms": info["ms"],
            "pairs": pairs}


def run_reference_arm(args, w, pts):
    """--impl reference: the reference's own code path (oracle/_ref), timed per
    call on the host cores; every step is a bounded sample of the workload."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from oracle import Reference
    ref = Reference()
    cores = ref.hw_threads()
    ds = ref.dataset(pts)
    # bound each step so (warmup + steps) finishes in a few minutes
    budget = max(1.0, 150.0 / max(1, args.steps + args.warmup))
    draws_s = _ref_calibrate(ref, ds, w, budget)
    rate = w.rate if draws_s >= w.draws else _ref_rate(w, draws_s)
    times, pairs = [], None
    for i in range(args.warmup + args.steps):
        _, _, info = ref.sng_dbscan(ds, w.eps, w.min_pts, rate, w.seed, threads=0)
        pairs = info["distance_evals"]
        if i >= args.warmup:
            times.append(info["ms"])
    ms = sum(times) / len(times)
    value = pairs / (ms / 1e3)
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (seeded generator, BASELINE.json shape)",
            "impl": "reference",
            "config": _workload_config(w, args.gpus, {
                "parallelism": f"{cores} host threads (reference std::thread workers)",
                "sample": _sample_desc(w, draws_s), "sample_draws": draws_s}),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "reference",
                             "sample": _sample_desc(w, draws_s)},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def relaunch_cmd(argv: list[str], gpus: int, port: int) -> list[str]:
    """`bench.py --gpus N` outside torchrun: the same command as N ranks."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
            f"--nproc-per-node={gpus}", "--master-addr", "127.0.0.1",
            f"--master-port={port}", os.path.abspath(__file__), *argv]


def _free_port() -> int:
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one rank per GPU: re-launch this command under torchrun (NCCL over NVLink)
        sys.exit(subprocess.call(relaunch_cmd(sys.argv[1:], args.gpus, _free_port())))
    rank, world, local = dist_env()
    if world != args.gpus and rank == 0:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; measuring {world} ranks",
              file=sys.stderr)
    from paper_2006_06743_b200 import synthetic
    w = synthetic.CONFIGS[args.config]

    if args.impl == "reference":
        if rank == 0:
            pts = synthetic.generate(args.config)
            run_reference_arm(args, w, pts)
        return

    import torch
    import torch.distributed as dist

    import paper_2006_06743_b200 as sng
    from paper_2006_06743_b200 import _lib
    from paper_2006_06743_b200.distributed import sng_dbscan_sharded

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    pts = synthetic.generate(args.config)  # same seeded bytes on every rank
    n, d = pts.shape
    pairs = n * w.draws
    host = torch.from_numpy(pts).pin_memory()
    points = host.to(dev, non_blocking=False)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step_device():
        if world == 1:
            return sng.sng_dbscan_device(points, w.eps, w.min_pts, w.rate, w.seed, timing=True)
        labels, roles, st = sng_dbscan_sharded(points, w.eps, w.min_pts, w.rate, w.seed)
        return labels, roles, st["edge_info"]

    # ---- warmup ----
    for _ in range(args.warmup):
        step_device()
    torch.cuda.synchronize(dev)

    # ---- timed device-resident steps ----
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    gather_ms, gather_bytes, gather_pairs, launches, lib_launches = [], 0, 0, 0, 0
    filter_bits = 32
    stage = {}
    info = None
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    dev_labels = dev_roles = None
    for k in range(args.steps):
        flush.zero_()  # L2 flush (outside the events)
        ev[k][0].record(stream)
        dev_labels, dev_roles, info = step_device()
        ev[k][1].record(stream)
        gather_ms.append(info.ms_gather)
        gather_bytes = info.gather_bytes
        filter_bits = getattr(info, "filter_bits", 32) or 32
        gather_pairs = info.gather_pairs
        launches += info.kernel_launches
        lib_launches += info.library_launches
        for nm in ("ms_sample", "ms_gather", "ms_extras", "ms_sort", "ms_cluster", "ms_total"):
            stage.setdefault(nm, []).append(getattr(info, nm))
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    clocks.stop()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    total_ms = sum(step_ms)
    if world > 1:
        t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    value = pairs / (ms_per_step / 1e3)

    # ---- e2e through the public host API (pinned host buffers) ----
    e2e = e2e_pageable = None
    if not args.no_e2e:
        labels_h = torch.empty(n, dtype=torch.int32).pin_memory()
        roles_h = torch.empty(n, dtype=torch.uint8).pin_memory()
        import ctypes as C
        L = _lib.lib()
        o = _lib.SngbOpts(local, 0, C.c_void_p(stream.cuda_stream), 0, 0)
        gi = _lib.SngbInfo()
        if world > 1:
            from paper_2006_06743_b200.distributed import shard_bounds
            chunk = (n + world - 1) // world
            rb_, re_ = shard_bounds(n, world, rank)
            shard_in = torch.zeros((chunk, d), dtype=torch.float32, device=dev)
            replica = torch.empty((chunk * world, d), dtype=torch.float32, device=dev)

        def step_e2e(src=None):
            if world == 1:
                # src: the pageable numpy array (what the Python / C++ mirrors pass)
                ptr = (src.ctypes.data_as(C.POINTER(C.c_float)) if src is not None
                       else C.cast(host.data_ptr(), C.POINTER(C.c_float)))
                rc = L.sngb_dbscan_f32(ptr, n, d,
                                       w.eps, w.min_pts, w.rate, w.seed, C.byref(o),
                                       C.cast(labels_h.data_ptr(), C.POINTER(C.c_int32)),
                                       C.cast(roles_h.data_ptr(), C.POINTER(C.c_uint8)),
                                       C.byref(gi))
                sng._check(rc)
            else:
                # replica: every rank uploads its own row shard over its PCIe link,
                # then one NCCL all-gather over NVLink assembles the full table
                shard_in[: re_ - rb_].copy_(host[rb_:re_], non_blocking=True)
                dist.all_gather_into_tensor(replica, shard_in)
                lab, rol, _ = sng_dbscan_sharded(replica[:n], w.eps, w.min_pts, w.rate, w.seed)
                if rank == 0:
                    labels_h.copy_(lab, non_blocking=True)
                    roles_h.copy_(rol, non_blocking=True)
                torch.cuda.current_stream(dev).synchronize()

        for _ in range(max(1, args.warmup)):
            step_e2e()
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        e_ms = []
        for _ in range(max(3, args.steps // 2)):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            step_e2e()
            b.record(stream)
            b.synchronize()
            e_ms.append(a.elapsed_time(b))
        e_tot = sum(e_ms)
        if world > 1:
            t = torch.tensor([e_tot], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e_tot = float(t.item())
        e_step = e_tot / len(e_ms)
        # the host call's results are the device-resident run's, bit for bit
        same = True
        if rank == 0:
            same = (torch.equal(labels_h, dev_labels.cpu()) and
                    torch.equal(roles_h, dev_roles.cpu()))
            if not same:
                raise SystemExit("bench.py: e2e labels/roles differ from the device-resident run")
        e2e = {"value": pairs / (e_step / 1e3), "unit": UNIT, "ms_per_step": e_step,
               "h2d_bytes_per_step": n * d * 4, "d2h_bytes_per_step": n * 4 + n * 1,
               "source": "pinned host memory (torch pin_memory)",
               "labels_equal_device_run": same}
        if world == 1 and not args.no_pageable:
            # pageable: the numpy array as the Python / C++ mirrors hand it over
            step_e2e(pts)
            torch.cuda.synchronize(dev)
            p_ms = []
            for _ in range(max(2, args.steps // 4)):
                flush.zero_()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                step_e2e(pts)
                b.record(stream)
                b.synchronize()
                p_ms.append(a.elapsed_time(b))
            if not (torch.equal(labels_h, dev_labels.cpu()) and
                    torch.equal(roles_h, dev_roles.cpu())):
                raise SystemExit("bench.py: pageable e2e labels differ from the device run")
            pm = statistics.mean(p_ms)
            e2e_pageable = {"value": pairs / (pm / 1e3), "unit": UNIT, "ms_per_step": pm,
                            "h2d_bytes_per_step": n * d * 4,
                            "d2h_bytes_per_step": n * 4 + n * 1,
                            "source": "pageable host memory (numpy)", "steps": len(p_ms)}

    # ---- roofline of the gather kernel ----
    peak, peak_kind = load_peaks()
    g_ms = statistics.mean(gather_ms) if gather_ms else 0.0
    # Narrow rows run the Floyd kernel concurrently with the gather (the step is
    # shorter), so the gather's in-step duration includes sharing the SMs; the
    # roofline uses the kernel alone, timed the same way over a few extra calls
    # with the overlap switched off (both durations are reported).
    g_ms_overlapped = None
    overlapped = world == 1 and (d <= 2 or (d + 3) // 4 * 4 <= 64) and n >= 10000
    if overlapped and g_ms > 0:
        old = os.environ.get("SNGB_OVERLAP")
        os.environ["SNGB_OVERLAP"] = "0"
        try:
            iso = []
            for _ in range(3):
                flush.zero_()
                _, _, inf = step_device()
                iso.append(inf.ms_gather)
            torch.cuda.synchronize(dev)
        finally:
            if old is None:
                del os.environ["SNGB_OVERLAP"]
            else:
                os.environ["SNGB_OVERLAP"] = old
        g_ms_overlapped, g_ms = g_ms, statistics.mean(iso)
    achieved = gather_bytes / (g_ms / 1e3) / 1e9 if g_ms > 0 else None
    q8 = filter_bits == 8
    head = filter_bits == 16  # sngb_head.cu: 4-byte head for every pair, fp32 row for survivors
    q8_split = q8 and (d + 15) // 16 + 1 >= Q8_SPLIT_MIN_RW  # head/tail gather (k_gather_q8s)
    bpp = gather_bytes / gather_pairs if gather_pairs else 4 * d  # algorithmic bytes per pair
    kname = ("k_gather_q8s" if q8_split else "k_gather_q8") if q8 else (
        "k_gather_head" if head else "k_gather")
    roofline = {"kernel": kname, "achieved": achieved, "unit": "GB/s",
                "traffic": load_traffic(w.name + ("_q8" if q8 else ("_head" if head else ""))),
                "algorithmic_bytes_per_launch": gather_bytes,
                "bytes_per_pair": bpp, "pairs_per_launch": gather_pairs,
                "filter": ("8-bit exact filter: u8 rows + norm, DP4A integer distances, "
                           "integer accept/reject thresholds, fp64 recheck in the band"
                           + ("; exact early reject on the 240-value head, survivors read "
                              "the tail" if q8_split else ""))
                if q8 else (("exact reject on a 2-byte head (two 8-bit coordinates, L2-resident); "
                             if (getattr(info, "head_bytes", 4) or 4) == 2 else
                             "exact reject on a 4-byte head (two 16-bit or four 8-bit coordinates, "
                             "L2-resident); ")
                            + "survivors: fp32 rows, fp32 guard band, fp64 recheck in the band"
                            if head else "fp32 rows, fp32 guard band, fp64 recheck in the band"),
                "kernel_ms": g_ms,
                "kernel_ms_in_step": g_ms_overlapped if g_ms_overlapped is not None else g_ms,
                "kernel_ms_note": ("kernel alone (SNGB_OVERLAP=0, 3 extra calls); in the step it "
                                   "shares the SMs with the Floyd kernel")
                if g_ms_overlapped is not None else "kernel in the timed steps",
                "kernel_share_of_step": (g_ms / ms_per_step) if ms_per_step else None}
    # The gather's real ceiling is the memory level the partner rows come from:
    # L2 when the row table (fp32 padded, or the 8-bit rows), or one L2-blocked
    # phase of it, is resident (the measured lean random-row gather of this row
    # shape), HBM otherwise (the measured copy peak: random 128-byte rows are
    # whole DRAM bursts, and our gather measured above the lean kernel there).
    row_bytes = (16 * ((d + 15) // 16 + 1)) if q8 else (16 if d == 3 else 4 * d)
    phased = d >= 256 and n * row_bytes > 100 * 2**20  # L2-blocked: one slice resident
    resident = n * row_bytes <= 100 * 2**20 or (phased and n * row_bytes <= 16 * 63 * 2**20)
    case, rows_per_s = load_gather_ceiling(
        d, min(n, int(63 * 2**20 // row_bytes)) if phased else n, row_bytes if q8 else None)
    l2_peak = rows_per_s * bpp / 1e9 if (resident and rows_per_s) else None
    if q8_split and resident and rows_per_s and gather_pairs:
        # every pair reads its 256-B head, a fraction f of them the rest of the
        # row: the ceiling is the time-weighted mix of the two measured gathers
        hcase, heads_per_s = load_gather_ceiling(d, n, row_bytes, Q8_HEAD_BYTES)
        head_alg = Q8_HEAD_VALS + 4
        f = max(0.0, (bpp - head_alg) / (d - Q8_HEAD_VALS + 4))
        roofline["tail_fraction"] = f
        if heads_per_s:
            l2_peak = bpp / (1.0 / heads_per_s + f / rows_per_s) / 1e9
            case = f"{hcase} + {case}"
        else:
            l2_peak = None
    if head and gather_pairs:
        # every pair reads its 2/4-byte head (L2), a fraction f its fp32 row (L2 or
        # HBM by table size), each at the measured random-row rate of its table
        hb = getattr(info, "head_bytes", 4) or 4
        roofline["head_bytes"] = hb
        hcase, heads_per_s = load_head_ceiling(n, hb)
        rcase, frows_per_s = load_gather_ceiling(d, n)
        f = max(0.0, (bpp - hb) / (4 * d))
        roofline["tail_fraction"] = f
        if heads_per_s and frows_per_s:
            # heads come from L2; survivors' rows from L2 too when the fp32 table
            # fits it (one resource: the times add), from HBM otherwise (two
            # resources working concurrently: the slower one bounds)
            t_head, t_rows = 1.0 / heads_per_s, f / frows_per_s
            rows_in_hbm = n * 4 * ((d + 3) // 4) > 100 * 2**20
            t_pair = max(t_head, t_rows) if rows_in_hbm else t_head + t_rows
            l2_peak = bpp / t_pair / 1e9
            case = f"{hcase} {'max' if rows_in_hbm else '+'} {rcase}"
            roofline["ceiling_model"] = ("max(head time, survivor-row time): L2 and HBM in "
                                         "parallel" if rows_in_hbm else
                                         "head time + survivor-row time: both from L2")
            resident = True
    eff = l2_peak if resident else peak
    # the fraction that means something: the kernel's own algorithmic bytes (what it
    # must read: heads + survivor rows, or 8-bit heads + tails, or fp32 rows) against
    # the measured random-gather ceiling of the memory level those rows come from
    roofline.update({
        "bound": "l2" if resident else "hbm",
        "bound_detail": ("l2 heads + survivor rows" if head else "l2 (random rows)")
        if resident else "hbm (random rows)",
        "peak": eff,
        "peak_source": (f"{case} in profiles/r01_gather_ceilings.jsonl "
                        "(tools/gather_ceiling.cu: lean random-row gather, measured on B200), "
                        "in the kernel's algorithmic bytes")
        if resident else f"MEASURED_PEAKS.json hbm_gbs ({peak_kind})",
        "frac": (achieved / eff) if (achieved and eff) else None,
        "hbm_gbs": peak,
        "concurrent_with": ("the Floyd kernel on a side stream (in the step)" if overlapped
                            else None)})
    # SURVEY 8(d)'s figure: 4*d bytes per pair (one fp32 partner row) -- an effective
    # rate against the HBM copy peak, not a roofline: the filters read far fewer bytes
    if g_ms > 0 and gather_pairs:
        a8 = 4.0 * d * gather_pairs / (g_ms / 1e3) / 1e9
        roofline["frac_8d"] = {
            "achieved": a8, "peak": peak, "unit": "GB/s", "value": a8 / peak,
            "note": "effective rate: 4*d B per pair (SURVEY 8(d)) / kernel time / "
                    "MEASURED_PEAKS hbm_gbs; > 1 means the filter avoided reading most rows"}
    ncu = load_ncu(w.name)
    if ncu:
        roofline["ncu"] = ncu
    # Two more bounds the gather is held against: the draws it
    # regenerates against the measured RNG throughput (tools/microbench.cu
    # rng_draw), and for rows narrower than an L2 sector (32 B) the share of
    # each fetched sector that is algorithmic bytes.
    rng_peak = None
    try:
        mb_path = os.path.join(ROOT, "profiles", "r02_microbench.jsonl")  # the current draw code
        if not os.path.exists(mb_path):
            mb_path = os.path.join(ROOT, "profiles", "r01_microbench.jsonl")
        for ln in open(mb_path):
            rec = json.loads(ln)
            if rec.get("bench") == "rng_draw":
                rng_peak = rec["draws_per_s"]
    except Exception:
        pass
    if g_ms > 0 and gather_pairs:
        draws_s = gather_pairs / (g_ms / 1e3)
        roofline["rng"] = {"draws_per_s": draws_s, "ceiling_draws_per_s": rng_peak,
                           "frac": (draws_s / rng_peak) if rng_peak else None,
                           "source": "profiles/" + os.path.basename(mb_path) + " rng_draw (one SplitMix64 + "
                                     "Lemire draw per lane, no memory traffic)"}
    if not q8 and not head and 4 * d < 32:
        row = 8 if d <= 2 else 16
        roofline["sector_efficiency"] = {"row_bytes": row, "algorithmic_bytes": 4 * d,
                                         "sector_bytes": 32, "frac": 4 * d / 32}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline(pts, w, args.cpu_budget_s)
        except Exception as e:  # the checker is optional; report why
            cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"unavailable: {e}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64-exact",
            "filter": roofline["filter"],
            "data": "synthetic (seeded generator, BASELINE.json shape)",
            "config": _workload_config(w, world, {
                "merge": "fixed-point union-find over NCCL all-reduce" if world > 1 else None,
                "replica": "row-shard upload + NCCL all-gather" if world > 1 else None}),
            "dtype_note": "decisions are the reference's fp64 decisions, bit for bit: "
                          "narrow filters (8-bit heads / rows, fp32 with a guard band) reject "
                          "or accept only where their error bound proves the fp64 result, "
                          "everything else is re-evaluated in fp64 in the reference's order",
            "e2e": e2e,
            "e2e_pageable": e2e_pageable,
            "gpu_launches": launches,
            "library_launches": lib_launches,
            "roofline": roofline,
            "cpu_baseline": cpu,
            "clocks": clocks.summary(),
            "stages_ms": {k: statistics.mean(v) for k, v in stage.items()},
            "result": {"edges": info.edges, "clusters": info.cluster_count,
                       "core": info.core_count, "border": info.border_count,
                       "noise": info.noise_count, "band_rechecks": info.band_rechecks,
                       "band_1e6": info.band_1e6, "fp32_flips": info.fp32_flips,
                       "collisions": info.collisions,
                       "irregular_vertices": info.irregular_vertices} if world == 1 else None,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
