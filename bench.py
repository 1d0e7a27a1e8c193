#!/usr/bin/env python
"""Falcon B200 benchmark -- one JSON line per run (driver contract).

Workload (BASELINE.json configs[1], "cfg2"): 256 Mi float64 values per GPU, a 2-decimal
random walk with 1 % injected outliers (synth kind outlier_injected, period 100, spike
3575 units, step 127; reference generator synthetic.hpp:36-115), default geometry
chunk_n = 1025, batch_values = 4,198,400 (pipeline.hpp:70-72).

One step = one pass of the hot path over the workload: device-resident compress of the
values into a .fln archive, then decompress of that archive back to values (both through
the C ABI, inputs resident in HBM).  value = uncompressed bytes / step time, summed over
GPUs.  e2e = the same round trip through falcon_compress_host / falcon_decompress_host
from pinned host buffers (H2D + D2H inside the timed region).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "compress/decompress GB/s (device-resident, 1/2/4/8 B200) and compression ratio"
CHUNK_N = 1025
BATCH_VALUES = 1025 * 1024 * 4
WORKLOADS = {
    # name: (kind, precision, values per GPU, decimal places, description)
    "cfg2": ("outlier", 0, 268_435_456, 2,
             "cfg2: 256Mi-value float64 random walk, 2 dp, 1% injected outliers "
             "(period 100, spike 3575 units, step 127)"),
    "cfg3": ("mixed", 1, 536_870_912, 0,
             "cfg3: 512Mi-value float32 reflecting walk, 1-6 dp drawn per 1025-value block"),
    "cfg1": ("walk", 0, 1_000_000, 2, "cfg1: 1M-value float64 random walk, 2 dp, step 127"),
}
FALLBACK_HBM = 6650.0


def hbm_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:  # noqa: BLE001
        return FALLBACK_HBM, "fallback"


def gen_values(kind, prec, n, dp, seed, out):
    from paper_2511_04140_b200 import synth
    return synth(kind, n, prec, dp=dp, seed=seed, period=100, units=3575, step=127, block=CHUNK_N, out=out)


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled while the timed region runs."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.path = tempfile.mktemp(suffix=".csv")

    def start(self):
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:  # noqa: BLE001
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:  # noqa: BLE001
            self.proc.kill()
        self.f.close()
        rows = []
        with open(self.path) as f:
            for line in f:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) >= 9:
                    rows.append(parts)
        os.unlink(self.path)
        if not rows:
            return None
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def link_bandwidth(torch, dev, host_pinned):
    """Pinned host<->device copy bandwidth (bytes/s), best of 3, CUDA events."""
    n = min(host_pinned.numel(), (1 << 30) // host_pinned.element_size())
    h = host_pinned[:n]
    d = torch.empty_like(h, device=dev)
    best = [0.0, 0.0]
    for _ in range(3):
        for k, (dst, src) in enumerate(((d, h), (h, d))):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            dst.copy_(src, non_blocking=True)
            e1.record()
            torch.cuda.synchronize()
            best[k] = max(best[k], h.numel() * h.element_size() / (e0.elapsed_time(e1) / 1e3))
    del d
    return best[0], best[1]


def cpu_reference_round_trip(values: np.ndarray, steps: int, warmup: int):
    """The unmodified reference (oracle/_ref) compress_pipeline + decompress_pipeline on
    host cores; falls back to the C restatement (single thread) if _ref is absent."""
    from oracle.oracle import Oracle, Ref, ref_available
    if ref_available():
        ref = Ref()
        cores = ref.threads()
        kind = "reference"

        def rt():
            a = ref.compress_pipeline(values, CHUNK_N, BATCH_VALUES, 16, 0)
            ref.decompress_pipeline(a, 0 if values.dtype == np.float64 else 1, 16, 0)
            return len(a)
    else:
        orc = Oracle()
        cores = 1
        kind = "port"

        def rt():
            a = orc.compress_archive(values, CHUNK_N, BATCH_VALUES)
            orc.decompress_archive(a, 0 if values.dtype == np.float64 else 1)
            return len(a)
    for _ in range(warmup):
        rt()
    times = []
    nbytes = 0
    for _ in range(steps):
        t0 = time.perf_counter()
        nbytes = rt()
        times.append(time.perf_counter() - t0)
    return kind, cores, times, nbytes


def run_reference(args, rank, world):
    if rank != 0:
        return
    kind, prec, n, dp, desc = WORKLOADS[args.workload]
    sample_n = min(n, args.cpu_sample_batches * BATCH_VALUES)
    vals = np.empty(sample_n, np.float64 if prec == 0 else np.float32)
    gen_values(kind, prec, sample_n, dp, 1, vals)
    kindname, cores, times, nbytes = cpu_reference_round_trip(vals, args.steps, args.warmup)
    t = sum(times)
    value = vals.nbytes * len(times) / t / 1e9
    sample = (f"first {sample_n} values ({sample_n // BATCH_VALUES} batches) of the {args.workload} "
              f"workload per step; compress_pipeline + decompress_pipeline, n_streams 16, all host threads")
    line = {
        "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * t / len(times), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64" if prec == 0 else "f32",
        "data": "synthetic", "impl": "reference",
        "config": {"workload": desc, "chunk_n": CHUNK_N, "batch_values": BATCH_VALUES,
                   "sample_values": sample_n, "ratio": nbytes / vals.nbytes},
        "cpu_baseline": {"value": value, "unit": "GB/s", "cores": cores, "kind": kindname, "sample": sample},
        "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    from paper_2511_04140_b200 import Codec, compress_bound, options, read_header

    kind, prec, n, dp, desc = WORKLOADS[args.workload]
    tdt = torch.float64 if prec == 0 else torch.float32
    esz = 8 if prec == 0 else 4
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    codec = Codec(local_rank)

    host_vals = torch.empty(n, dtype=tdt, pin_memory=True)
    gen_values(kind, prec, n, dp, 1 + rank, host_vals.numpy())
    d_vals = host_vals.to(dev)
    cap = compress_bound(prec, n, CHUNK_N, BATCH_VALUES)
    d_arc = torch.empty(cap, dtype=torch.uint8, device=dev)
    d_back = torch.empty(n, dtype=tdt, device=dev)
    stream = torch.cuda.current_stream(dev)
    sh = stream.cuda_stream

    d_nb = torch.zeros(1, dtype=torch.int64, device=dev)   # archive length, device-resident

    def step(evs=None, chained=True):
        """One pass of the hot path: compress the workload, then decompress the archive.
        The timed steps chain the two on the stream with no host round trip (the archive
        length stays on the device); device errors are collected by codec.sync()."""
        if evs is not None:
            codec.set_kernel_events(enc=(evs[0], evs[1]), dec=(evs[2], evs[3]))
        if not chained:
            _, nb = codec.compress_device(d_vals, CHUNK_N, BATCH_VALUES, out=d_arc, stream=sh)
            codec.decompress_device(d_arc, nb, out=d_back, stream=sh)
            return nb
        codec.compress_device_async(d_vals, d_arc, d_nb, CHUNK_N, BATCH_VALUES, stream=sh)
        if world > 1:
            # the one exchange step of a sharded archive: every rank's byte total, so
            # shard g lands at 47 + sum_{h<g} (bytes_h - 47) when concatenated
            sizes = torch.zeros(world, dtype=torch.int64, device=dev)
            sizes[rank] = d_nb[0]
            dist.all_reduce(sizes)
        codec.decompress_device_chained(d_arc, d_nb, info, d_back, stream=sh)
        return None

    # correctness gate before timing: round trip must be bit-exact (synchronous API)
    nb = step(chained=False)
    torch.cuda.synchronize()
    info = read_header(d_arc[:47].cpu().numpy().tobytes())
    assert torch.equal(d_back.view(torch.int64 if prec == 0 else torch.int32),
                       d_vals.view(torch.int64 if prec == 0 else torch.int32)), "round trip mismatch"
    ratio = nb / (n * esz)
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    kev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.steps)]
    for evs in kev:          # torch creates the CUDA event lazily on first record
        for e in evs:
            e.record(stream)
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    clocks = ClockSampler(local_rank)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    time.sleep(0.2)
    t0.record(stream)
    for k in range(args.steps):
        step(kev[k])
    t1.record(stream)
    torch.cuda.synchronize()
    codec.sync(sh)   # raises on any device-side error of the timed steps
    assert int(d_nb.item()) == nb, "chained steps produced a different archive length"
    if world > 1:
        dist.barrier()
    time.sleep(0.1)
    clk = clocks.stop()
    codec.set_kernel_events()
    elapsed = t0.elapsed_time(t1) / 1e3
    enc_ms = [e[0].elapsed_time(e[1]) for e in kev]
    dec_ms = [e[2].elapsed_time(e[3]) for e in kev]
    if world > 1:
        t = torch.tensor([elapsed], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed = float(t.item())
    in_bytes = n * esz
    value = world * in_bytes * args.steps / elapsed / 1e9

    # ---- e2e through the host-buffer C ABI (pinned H2D / D2H inside the timed region) ----
    e2e = None
    if not args.no_e2e:
        h_arc = torch.empty(cap, dtype=torch.uint8, pin_memory=True)
        h_back = torch.empty(n, dtype=tdt, pin_memory=True)
        opt = options(CHUNK_N, BATCH_VALUES, 16, 0)
        hv, ha, hb = host_vals.numpy(), h_arc.numpy(), h_back.numpy()

        def e2e_step():
            a = codec.compress_host(hv, opt, out=ha)
            codec.decompress_host(a, prec, opt, out=hb)
            return len(a)

        nb_e = e2e_step()
        assert nb_e == nb and hb.view(np.uint8).tobytes()[:4096] == hv.view(np.uint8).tobytes()[:4096]
        times = []
        for _ in range(args.e2e_steps):
            if world > 1:
                dist.barrier()
            s = time.perf_counter()
            e2e_step()
            times.append(time.perf_counter() - s)
        te = sum(times)
        if world > 1:
            t = torch.tensor([te], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            te = float(t.item())
        e2e = {"value": world * in_bytes * len(times) / te / 1e9, "unit": "GB/s",
               "h2d_bytes_per_step": in_bytes + nb_e, "d2h_bytes_per_step": nb_e + in_bytes,
               "ms_per_step": 1e3 * te / len(times)}
        # the host link bounds this number: pinned copy bandwidth measured on this box, and
        # the fraction of the link-bound time (compress: H2D of values || D2H of the
        # archive, then decompress: H2D of the archive || D2H of values) achieved
        h2d, d2h = link_bandwidth(torch, dev, host_vals)
        bound_s = max(in_bytes / h2d, nb_e / d2h) + max(nb_e / h2d, in_bytes / d2h)
        e2e.update({"link_h2d_gbs": h2d / 1e9, "link_d2h_gbs": d2h / 1e9,
                    "link_frac": bound_s / (te / len(times))})
        del h_arc, h_back

    if rank != 0:
        return
    peak, peak_kind = hbm_peak()
    algo = in_bytes + nb   # sizeof(T) * (1 + ratio) per value, both directions
    enc_avg, dec_avg = statistics.mean(enc_ms) / 1e3, statistics.mean(dec_ms) / 1e3
    dom = "encode" if enc_avg >= dec_avg else "decode"
    dom_t = max(enc_avg, dec_avg)
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(prof):
        try:
            with open(prof) as f:
                traffic = json.load(f).get(f"{args.workload}_{dom}")
        except Exception:  # noqa: BLE001
            traffic = None
    roofline = {"bound": "hbm", "achieved": algo / dom_t / 1e9, "peak": peak, "unit": "GB/s",
                "frac": algo / dom_t / 1e9 / peak, "traffic": traffic, "kernel": f"{dom}_chunks_kernel",
                "peak_source": f"{peak_kind} hbm_gbs (MEASURED_PEAKS.json)" if peak_kind == "measured"
                else "fallback 6650 GB/s (B200_PROFILING.md)",
                "encode_kernel_ms": 1e3 * enc_avg, "decode_kernel_ms": 1e3 * dec_avg,
                "encode_frac": algo / enc_avg / 1e9 / peak, "decode_frac": algo / dec_avg / 1e9 / peak}
    cpu = None
    if world == 1 and not args.no_cpu:
        sample_n = min(n, args.cpu_sample_batches * BATCH_VALUES)
        kindname, cores, times, _ = cpu_reference_round_trip(host_vals.numpy()[:sample_n], 2, 1)
        cpu = {"value": sample_n * esz * len(times) / sum(times) / 1e9, "unit": "GB/s", "cores": cores,
               "kind": kindname,
               "sample": f"first {sample_n} values ({sample_n // BATCH_VALUES} batches) of the workload; "
                         f"compress_pipeline + decompress_pipeline round trip, median of 2 after 1 warm-up"}
    line = {
        "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * elapsed / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64" if prec == 0 else "f32",
        "data": "synthetic (counter-free mt19937_64 reference generator, seed 1+rank)",
        "config": {"workload": desc, "values_per_gpu": n, "chunk_n": CHUNK_N, "batch_values": BATCH_VALUES,
                   "ratio": ratio, "archive_bytes_per_gpu": nb,
                   "compress_gbs": world * in_bytes / statistics.mean(enc_ms) * 1e3 / 1e9,
                   "decompress_gbs": world * in_bytes / statistics.mean(dec_ms) * 1e3 / 1e9,
                   "l2": f"inputs {in_bytes / 1e9:.2f} GB per GPU exceed the 126 MB L2; no flush",
                   "parallelism": f"dp{world} (independent batch-range shards; NCCL all_reduce of "
                                  f"archive byte totals for shard placement)" if world > 1 else "dp1"},
        "roofline": roofline,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": 4 * args.steps,   # encode, place, walker, decode
        "clocks": clk,
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="cfg2")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--cpu-sample-batches", type=int, default=8)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
