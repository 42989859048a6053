#!/usr/bin/env python
"""Benchmark: Chung–Lu edges/sec on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4]
                    [--impl ours|reference] [--mode counter|reference]

One step = one pass of the generator over the whole workload (every source
node of this rank's UCP partition): the device plan + the sampler with its
fused fold (streaming configs) or count+scan+write (materialised configs).
Multi-GPU: launched by torchrun, one process per GPU; each rank generates its
UCP partition (weak-free strong split of one graph; see `scaling`).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "CL edges/sec at 1/2/4/8 B200 (n=1e9, avg deg 500); % of HBM-write roofline"
UNIT = "edges/s"
BYTES_PER_EDGE = 8  # two uint32 node ids (the algorithmic write per edge)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c4", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--num-vertices", dest="n", type=int, default=None,
                    help="override the node count (testing only)")
    ap.add_argument("--mode", default="counter", choices=["reference", "counter"],
                    help="random stream of the streaming configs (materialised C1/C2 always "
                         "use the bit-exact reference stream)")
    ap.add_argument("--track-shift", type=int, default=6)
    ap.add_argument("--ring-log2", type=int, default=28)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    return ap.parse_args()


# --------------------------------------------------------------------------- util
def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # wait until nvidia-smi is up (its start-up is longer than a short timed
            # region), then drop that pre-region sample
            t0 = time.time()
            while not self.lines and time.time() - t0 < 5.0 and self.proc.poll() is None:
                time.sleep(0.01)
            self.lines.clear()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        at_end = False
        if not self.lines:
            # the timed region was shorter than the 200 ms sampling period: take the
            # first sample after it (GPU just left the region) and say so
            t0 = time.time()
            while not self.lines and time.time() - t0 < 1.0:
                time.sleep(0.005)
            at_end = bool(self.lines)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm),
                **({"sampled": "first sample after the timed region (region < 200 ms period)"}
                   if at_end else {})}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # test hook: map every rank to one GPU (multi-rank logic on a 1-GPU box, gloo)
    local = int(os.environ.get("CLGEN_DEVICE_OVERRIDE", local))
    return ws, rank, local


# --------------------------------------------------------------------------- CPU arm
def workload_config(name: str, n: int) -> dict:
    """The workload identity shared by both arms' JSON lines (same `config`)."""
    import inputs
    wl = inputs.WORKLOADS[name]
    return {"workload": f"{name}: {wl.desc}", "n": int(n), "seed": wl.seed,
            "materialised": wl.materialise}


PLAN_PARTS = 64  # plan_ucp_oracle(ws, 64): the sampling frame of SURVEY.md §8(d)


class CpuReference:
    """The reference CPU generator (oracle/_ref: the unmodified reference
    library, compiled from its own sources) on a bounded, extrapolated sample
    of the workload (SURVEY.md §8(d) "CPU baseline timing"):

    * plan_ucp_oracle(ws, 64) is built once (partition.cpp:159-203);
    * `cores` of its 64 UCP partitions, evenly spread, are sampled (all 64
      when the host has >= 64 cores); each contributes the prefix of the
      partition holding about `seconds` of single-thread work;
    * create_edges_range runs on those prefixes in parallel std::threads (the
      acceptance.cpp:221-254 per-partition pattern), count-only EdgeCounter;
    * value = sampled edges / wall time of the parallel section; the full
      workload time is extrapolated as m / value.
    Never imports the product package and never touches the GPU."""

    def __init__(self, w: np.ndarray, seconds: float):
        import oracle
        self.cores = os.cpu_count() or 1
        self.R = oracle.ref()
        t0 = time.time()
        self.ws = self.R.weight_sequence(w)
        S = self.ws.sum_S
        self.plan = self.R.plan_ucp_oracle(self.ws, PLAN_PARTS)
        self.plan_s = time.time() - t0
        # suffix-form expected edges per source (cost.cpp:62-77 minus the 1)
        # to size each prefix; a sizing aid only, the timing is the reference's
        cs = np.cumsum(w)
        e = w / S * (S - cs)
        ecum = np.cumsum(e)
        del cs, e
        self.m = float(ecum[-1])
        # per-thread rate probe (~0.2 s) at the median partition
        mid = PLAN_PARTS // 2
        lo = int(self.plan[mid])
        hi = self._prefix_end(ecum, lo, int(self.plan[mid + 1]), 1e6)
        tot, ms = self.R.parallel_ranges_count(self.ws, S, [(lo, hi)], 1)
        rate1 = max(tot / max(ms, 1e-3) * 1e3, 1e5)
        self.per_thread = rate1 * seconds
        k = min(self.cores, PLAN_PARTS)
        self.parts = sorted({int(round((i + 0.5) * PLAN_PARTS / k - 0.5)) for i in range(k)})
        self.ranges = []
        for i in self.parts:
            lo, end = int(self.plan[i]), int(self.plan[i + 1])
            self.ranges.append((lo, self._prefix_end(ecum, lo, end, self.per_thread)))
        self.sample_edges = float(sum(ecum[h - 1] - (ecum[l - 1] if l else 0.0)
                                      for l, h in self.ranges if h > l))
        del ecum

    @staticmethod
    def _prefix_end(ecum, lo, end, edges):
        base = ecum[lo - 1] if lo else 0.0
        hi = int(np.searchsorted(ecum, base + edges, side="right")) + 1
        return max(lo + 1, min(hi, end))

    def step(self, seed: int) -> dict:
        tot, ms = self.R.parallel_ranges_count(self.ws, self.ws.sum_S, self.ranges, seed)
        v = tot / (ms / 1e3)
        return {"value": v, "unit": UNIT, "cores": len(self.ranges), "kind": "reference",
                "extrapolated": True, "nproc": self.cores,
                "sample": (f"prefixes of {len(self.ranges)} of the {PLAN_PARTS} plan_ucp_oracle(ws,"
                           f"{PLAN_PARTS}) partitions (ids {self.parts[0]}..{self.parts[-1]}), "
                           f"~{self.per_thread:.3g} expected edges each, create_edges_range in "
                           f"{len(self.ranges)} parallel std::threads (nproc={self.cores}), "
                           f"count-only sink: {tot} edges in {ms / 1e3:.2f} s; full workload "
                           f"m={self.m:.4g} edges extrapolates to {self.m / v:.4g} s"),
                "plan_s": round(self.plan_s, 1)}


def cpu_baseline(w: np.ndarray, seed: int, seconds: float) -> dict:
    return CpuReference(w, seconds).step(seed)


def run_reference(args):
    """--impl reference: the unmodified reference (oracle/_ref) on the host
    cores.  Imports only `inputs` (input preparation) and `oracle` (the
    reference build); under torchrun only rank 0 works."""
    ws_, rank, _ = dist_env()
    if rank != 0:
        return
    import inputs
    w = inputs.make(args.config, args.n)
    seed = inputs.WORKLOADS[args.config].seed
    ref = CpuReference(w, args.cpu_seconds / 2)
    vals, step_ms, last = [], [], None
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        last = ref.step(seed + i)
        if i >= args.warmup:
            vals.append(last["value"])
            step_ms.append((time.perf_counter() - t0) * 1e3)
    v = float(np.median(vals))
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": float(np.mean(step_ms)),
        "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(args.config, w.size),
        "cpu_baseline": {**last, "value": v},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


def write_only_gbs(torch, stream) -> float | None:
    """Write-only HBM bandwidth on this box: best of 10
    fills of a 4 GiB buffer, CUDA events on the bench stream, outside the
    timed region.  Reported beside the copy-bandwidth peak."""
    try:
        with torch.cuda.stream(stream):
            buf = torch.empty(1 << 29, dtype=torch.int64, device="cuda")
            best = None
            for _ in range(10):
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                buf.fill_(1)
                e1.record(stream)
                e1.synchronize()
                ms = e0.elapsed_time(e1)
                best = ms if best is None or ms < best else best
            nbytes = buf.numel() * 8
            del buf
        return nbytes / (best / 1e3) / 1e9
    except Exception:
        return None


# --------------------------------------------------------------------------- GPU arm
def run_ours(args):
    import torch
    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    comm = None
    if world > 1:
        import torch.distributed as dist
        backend = os.environ.get("CLGEN_DIST_BACKEND", "nccl")  # gloo: multi-rank test on one GPU
        if backend == "nccl":
            # NCCL's own init log names the communicator size ("nranks")
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
        else:
            dist.init_process_group(backend)
        comm = {"backend": dist.get_backend(), "nranks": dist.get_world_size()}
        if backend == "nccl":
            v = torch.cuda.nccl.version()
            comm["nccl_version"] = ".".join(map(str, v)) if isinstance(v, tuple) else v
        print(f"[clgen] rank {rank}: {comm['backend']} communicator nranks={comm['nranks']}",
              file=sys.stderr, flush=True)
    import inputs
    from paper_1406_1215_b200 import api, runtime

    wl = inputs.WORKLOADS[args.config]
    seed = wl.seed
    t0 = time.time()
    w_host = runtime.shared_weights(args.config, args.n, world, rank, local)
    prep_s = time.time() - t0
    n = int(w_host.size)

    dev = api.Device(local)
    w_dev = torch.from_numpy(w_host).to(f"cuda:{local}")
    dev.set_weights(w_dev)
    del w_dev
    S = dev.blocked_sum()
    ws = api.WeightSequence(w_host, S, None, dev)
    bounds = runtime.plan(ws, world, rank)
    lo, hi = int(bounds[rank]), int(bounds[rank + 1])

    materialise = wl.materialise
    stream = dev.torch_stream()
    ring = None
    out = None
    if materialise:
        cap = int(runtime.expected_edges(w_host, S, lo, hi) * 1.01 + 1_000_000)
        out = torch.empty((cap, 2), dtype=torch.int32, device=f"cuda:{local}")
    else:
        ring = torch.empty((1 << args.ring_log2, 2), dtype=torch.int32, device=f"cuda:{local}")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{local}")
    small_inputs = n * 8 < (256 << 20)

    flags = [0]

    def step():
        if materialise:
            e, nf = api.create_edges_range(ws, S, lo, hi, seed, out=out, return_flagged=True)
            flags[0] = max(flags[0], int(nf))
            return int(e.shape[0])
        r = api.stream_range(ws, S, lo, hi, seed, mode=args.mode, track_shift=args.track_shift,
                             degree=deg, accumulate=False, ring=ring)
        flags[0] = max(flags[0], int(r.flagged))
        return r.count

    deg = None
    if not materialise:
        ntr = (n + (1 << args.track_shift) - 1) >> args.track_shift
        deg = torch.zeros(ntr, dtype=torch.int32, device=f"cuda:{local}")

    for _ in range(args.warmup):
        edges = step()
    torch.cuda.synchronize()

    clocks = ClockSampler(local)
    clocks.start()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    launches0 = dev.launch_count
    total_ms, kern_ms, edges_total = 0.0, 0.0, 0
    for _ in range(args.steps):
        if small_inputs:
            flush.zero_()  # L2 flush between timed iterations (inputs < L2)
            torch.cuda.synchronize()
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        edges = step()
        ev1.record(stream)
        ev1.synchronize()
        total_ms += ev0.elapsed_time(ev1)
        kern_ms += dev.last_kernel_ms()
        edges_total += edges
    launches = dev.launch_count - launches0
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    clk = clocks.stop()

    # the level-1 plan's per-rank device phases for an 8-GPU run, timed rank
    # by rank on this GPU (untimed for `value`; N = 1 plans trivially)
    plan8 = None
    if world == 1 and not materialise:
        plan8 = runtime.plan_phase_times(dev, n, S, 8)

    # level-2 balance evidence: one extra untimed step with per-warp busy intervals
    dev.set_warp_profile(True)
    step()
    wprof = dev.warp_profile()
    dev.set_warp_profile(False)

    # max over ranks of the device time; sum of edges
    ms_step = total_ms / args.steps
    per_gpu = [ms_step]
    planned = None
    if world > 1:  # planned cost per GPU (fill_partition_costs) beside the measured times
        pc = api.fill_partition_costs(api.PartitionPlan("ucp", world, n, np.asarray(bounds)), ws)
        planned = {"per_gpu_cost": pc.tolist(), "max_over_mean": float(pc.max() / pc.mean())}
    if world > 1:
        import torch.distributed as dist
        g = torch.zeros(world, dtype=torch.float64, device=runtime.comm_device(local))
        mine = torch.tensor([ms_step], dtype=torch.float64, device=runtime.comm_device(local))
        dist.all_gather_into_tensor(g, mine)
        per_gpu = g.cpu().tolist()
    if world > 1:
        import torch.distributed as dist
        cdev = runtime.comm_device(local)
        t = torch.tensor([ms_step, kern_ms / args.steps], dtype=torch.float64, device=cdev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e = torch.tensor([edges_total], dtype=torch.int64, device=cdev)
        dist.all_reduce(e)
        ms_step, kern_step = float(t[0]), float(t[1])
        edges_all = int(e[0]) // args.steps
        f = torch.tensor([flags[0]], dtype=torch.int64, device=cdev)
        dist.all_reduce(f)
        flags[0] = int(f[0])
    else:
        kern_step = kern_ms / args.steps
        edges_all = edges_total // args.steps
    value = edges_all / (ms_step / 1e3)

    # ---- e2e through the public API with host buffers -------------------
    e2e = None
    if not args.no_e2e:
        e2e = runtime.e2e_measure(args, w_host, world, rank, local, lo, hi, seed, materialise)

    hbm, peak_kind = peaks()
    write_gbs = write_only_gbs(torch, stream) if rank == 0 else None
    my_edges = edges_total // args.steps
    achieved = my_edges * BYTES_PER_EDGE / (kern_step / 1e3) / 1e9
    traffic = runtime.ncu_traffic(args.config, args.mode)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline(w_host, seed, args.cpu_seconds)
        except Exception as ex:  # the reference build may be absent on odd boxes
            cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"unavailable: {ex}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": workload_config(args.config, n),
            "run": {"edges_per_step": edges_all,
                       "stream_mode": args.mode if not materialise else "reference",
                       "materialised": materialise,
                       "track_shift": None if materialise else args.track_shift,
                       "ring_pairs": None if materialise else (1 << args.ring_log2),
                       "l2": "flushed (256 MB write) between timed steps" if small_inputs
                       else f"inputs larger than L2 ({n * 8 / 1e9:.1f} GB weights)",
                       "parallelism": f"ucp{world}", "weights_prep_s": round(prep_s, 1),
                       "weights_prep": ("device (clgen_dev_synth_powerlaw) + read-back" if args.config in runtime.DEVICE_RECIPES and os.environ.get("CLGEN_HOST_SYNTH", "0") != "1" else "host (inputs)")},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                         "frac": achieved / hbm, "traffic": traffic,
                         "peak_source": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs, copy)",
                         "kernel_ms": kern_step,
                         "write_only_gbs": write_gbs,
                         "frac_of_write_only": (achieved / write_gbs) if write_gbs else None,
                         "algorithmic_bytes": f"{BYTES_PER_EDGE} B/edge x {my_edges} edges"},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(launches),
            # sources whose skip ratio fell in the libm-ambiguity band (reference
            # stream only); the counter stream has none by construction
            "n_flagged": flags[0],
            "comm": comm,
            "plan_g8_on_one_gpu": plan8,
            "load_balance": {
                "per_launch_warp_busy": [
                    {"max_over_mean": round(p["max_over_mean"], 4), "mean_ms": round(p["mean_ms"], 3),
                     "max_ms": round(p["max_ms"], 3), "span_ms": round(p["span_ms"], 3),
                     "warps": p["warps"]} for p in wprof],
                "per_gpu_ms": per_gpu,
                "planned": planned,
                "per_gpu_max_over_mean": max(per_gpu) / (sum(per_gpu) / len(per_gpu))},
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
