#!/usr/bin/env python
"""Falcon B200 benchmark -- one JSON line per run (driver contract).

Workloads (BASELINE.json configs; default geometry chunk_n = 1025, batch_values =
4,198,400, pipeline.hpp:70-72):

  cfg1  1,000,000 f64, 2-dp random walk (reference generator, seed 1); the step is one
        CUDA-graph replay of the device-resident round trip (launch-bound size)
  cfg2  268,435,456 f64 per GPU, 2-dp walk with 1 % injected outliers (period 100, spike
        3575 units) -- the default; weak scaling under torchrun
  cfg3  536,870,912 f32, reflecting walk, 1-6 dp drawn per 1025-value block (pinned kind)
  cfg4  1,073,741,824 f64 (8 GiB), 2-dp walk, HOST-resident: e2e through the async
        H2D / kernel / D2H pipeline from pinned and from pageable buffers
  cfg5  8,589,934,592 f64 (64 GiB) counter-based field (csrc/field.cuh), strong scaling:
        rank g of G owns batches [g*B/G, (g+1)*B/G), generated on its own device

One step = device-resident compress of the workload into a .fln archive, then decompress
of that archive (both through the C ABI, chained on one stream, inputs resident in HBM).
value = uncompressed bytes / step time, summed over GPUs.  e2e = the same round trip
through the host-buffer entry points (falcon_compress_host / falcon_decompress_host) with
H2D + D2H inside the timed region.  The reference arm (--impl reference) runs the
unmodified reference library (oracle/_ref, the reference's own sources built in place)
on the host cores over the same workload.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--workload cfg1|cfg2|cfg3|cfg4|cfg5]
"""
from __future__ import annotations

import argparse
import hashlib
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
F64, F32 = 0, 1

WORKLOADS = {
    "cfg1": dict(kind="walk", prec=F64, n=1_000_000, dp=2, gen="reference", graph=True,
                 desc="cfg1: 1M-value float64 sensor random walk, 2 dp, step 127, seed 1"),
    "cfg2": dict(kind="outlier", prec=F64, n=268_435_456, dp=2, gen="reference",
                 desc="cfg2: 256Mi-value float64 random walk, 2 dp, 1% injected outliers "
                      "(period 100, spike 3575 units, step 127)"),
    "cfg3": dict(kind="mixed", prec=F32, n=536_870_912, dp=0, gen="pinned",
                 desc="cfg3: 512Mi-value float32 reflecting walk, 1-6 dp drawn per 1025-value block"),
    "cfg4": dict(kind="walk", prec=F64, n=1_073_741_824, dp=2, gen="reference", host=True,
                 desc="cfg4: 8 GiB host-resident float64 2-dp random walk through the async "
                      "H2D/compute/D2H pipeline"),
    "cfg5": dict(kind="field", prec=F64, n=8_589_934_592, dp=2, gen="device", strong=True,
                 desc="cfg5: 64 GiB float64 counter-based field (two triangle waves + noise, 2 dp), "
                      "sharded by batch range"),
}
FALLBACK_HBM = 6650.0
SEED = 1


def hbm_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured hbm_gbs (MEASURED_PEAKS.json)"
    except Exception:  # noqa: BLE001
        return FALLBACK_HBM, "fallback 6650 GB/s (B200_PROFILING.md)"


def dtype_of(prec):
    return np.float64 if prec == F64 else np.float32


def synth_kwargs(w, seed):
    return dict(dp=w["dp"], seed=seed, step=127, period=100, units=3575)


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
                                          "--format=csv,noheader,nounits", "-lms", "20"],
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


# --------------------------------------------------------------------------------------
# inputs: the reference's own generator (oracle/_ref synth::generator) where it has the
# kind, the oracle's pinned restatement otherwise.  Our arm uses the library's bit-equal
# twins (falcon_synth_fill), so both arms compress the same bytes.
def reference_values(w, n, seed, first=0):
    from oracle.oracle import Oracle, Ref, ref_available
    out = np.empty(n, dtype_of(w["prec"]))
    if w["kind"] in ("walk", "outlier") and ref_available():
        r = Ref()
        kw = synth_kwargs(w, seed)
        out[:] = r.synth(w["kind"], n, w["prec"], dp=kw["dp"], seed=seed, step=127, period=kw["period"],
                         units=kw["units"])
        return out
    Oracle().synth(w["kind"], n, w["prec"], dp=w["dp"], seed=seed, step=127, period=100, units=3575,
                   block=CHUNK_N, first=first, out=out)
    return out


def cpu_round_trip(values: np.ndarray, steps: int, warmup: int, decode_check=False):
    """compress_pipeline + decompress_pipeline of the unmodified reference (oracle/_ref) on
    all host threads; the C restatement (one thread) where _ref is absent."""
    from oracle.oracle import Oracle, Ref, ref_available
    prec = F64 if values.dtype == np.float64 else F32
    if ref_available():
        ref = Ref()
        cores, kind = ref.threads(), "reference"

        def rt():
            a = ref.compress_pipeline(values, CHUNK_N, BATCH_VALUES, 16, 0)
            ref.decompress_pipeline(a, prec, 16, 0)
            return a
    else:
        orc = Oracle()
        cores, kind = 1, "port"

        def rt():
            a = orc.compress_archive(values, CHUNK_N, BATCH_VALUES)
            orc.decompress_archive(a, prec)
            return a
    for _ in range(warmup):
        rt()
    times, arc = [], b""
    for _ in range(steps):
        t0 = time.perf_counter()
        arc = rt()
        times.append(time.perf_counter() - t0)
    return kind, cores, times, arc


def run_reference(args, rank, world):
    """--impl reference: the reference's CPU path on this box's host cores, rank 0 only."""
    if rank != 0:
        return
    w = WORKLOADS[args.workload]
    esz = 8 if w["prec"] == F64 else 4
    n = w["n"]
    cap = args.ref_max_values
    sample_n = n if n <= cap else (cap // BATCH_VALUES) * BATCH_VALUES
    vals = reference_values(w, sample_n, SEED)
    kind, cores, times, arc = cpu_round_trip(vals, args.steps, args.warmup)
    med = statistics.median(times)
    value = sample_n * esz / med / 1e9
    same = sample_n == n
    sample = (f"{'all' if same else 'first'} {sample_n} values ({(sample_n + BATCH_VALUES - 1) // BATCH_VALUES} "
              f"batches) of the {args.workload} workload per step; compress_pipeline + decompress_pipeline, "
              f"n_streams 16, {cores} host threads; median of {len(times)} steps after {args.warmup} warm-up")
    line = {
        "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * med, "higher_is_better": True,
        "scaling": "strong" if w.get("strong") else "weak", "vs_baseline": None,
        "dtype": "f64" if w["prec"] == F64 else "f32", "data": "synthetic", "impl": "reference",
        "config": {"workload": w["desc"], "chunk_n": CHUNK_N, "batch_values": BATCH_VALUES,
                   "values": sample_n, "same_config": same, "ratio": len(arc) / (sample_n * esz),
                   "archive_sha256_16": hashlib.sha256(arc).hexdigest()[:16],
                   "generator": "reference synth::generator (oracle/_ref)" if w["gen"] == "reference"
                   else "pinned kind, oracle restatement"},
        "cpu_baseline": {"value": value, "unit": "GB/s", "cores": cores, "kind": kind, "sample": sample},
        "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------------------
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


def our_launches_per_step(n_values, prec):
    """Kernels of one compress + decompress (csrc/encode.cu plan_waves, decode.cu): the
    chunk sampler, one encode launch per wave of batches + the final placement, then
    walker + decoder."""
    if n_values == 0:
        return 0
    nb = (n_values + BATCH_VALUES - 1) // BATCH_VALUES
    cpb = (BATCH_VALUES + CHUNK_N - 1) // CHUNK_N if nb > 1 else (n_values + CHUNK_N - 1) // CHUNK_N
    n_chunks = (nb - 1) * cpb + ((n_values - (nb - 1) * BATCH_VALUES) + CHUNK_N - 1) // CHUNK_N
    slot = 8320 if prec == F64 else 4224                     # encode_slot_bytes
    slots = int(os.environ.get("FALCON_ENC_RING_BYTES", str(4 << 30))) // slot
    wave = int(os.environ.get("FALCON_ENC_WAVE_CHUNKS", "0")) or (n_chunks if slots >= n_chunks
                                                                   else (slots - 128) // 2)
    wb = nb if wave >= n_chunks else max(1, min(wave // cpb, 65534, nb))
    return 1 + (nb + wb - 1) // wb + 1 + 2


def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    from paper_2511_04140_b200 import Codec, compress_bound, options, read_header, synth

    w = WORKLOADS[args.workload]
    prec = w["prec"]
    tdt = torch.float64 if prec == F64 else torch.float32
    idt = torch.int64 if prec == F64 else torch.int32
    esz = 8 if prec == F64 else 4
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    codec = Codec(local_rank)
    stream = torch.cuda.current_stream(dev)
    sh = stream.cuda_stream

    # ---- this rank's values: weak scaling (per-rank copy of the workload, seed 1 + rank)
    #      or strong scaling (rank's batch range of one global stream) ----
    if w.get("strong"):
        nb_total = (w["n"] + BATCH_VALUES - 1) // BATCH_VALUES
        b0, b1 = rank * nb_total // world, (rank + 1) * nb_total // world
        first = b0 * BATCH_VALUES
        n = min(b1 * BATCH_VALUES, w["n"]) - first
        seed = SEED
    else:
        first, n, seed = 0, w["n"], SEED + rank
    host_vals = None
    if w["gen"] == "device":
        d_vals = torch.empty(n, dtype=tdt, device=dev)
        codec.synth_device(d_vals, w["kind"], first=first, dp=w["dp"], seed=seed)
    else:
        host_vals = torch.empty(n, dtype=tdt, pin_memory=True)
        synth(w["kind"], n, prec, block=CHUNK_N, out=host_vals.numpy(), **synth_kwargs(w, seed))
        d_vals = host_vals.to(dev)
    torch.cuda.synchronize()
    in_bytes = n * esz
    # archive buffer: the worst-case bound, except for the 64 GiB shard where three full
    # copies would not fit one GPU (the field's ratio is ~0.127; a too-small buffer fails
    # loudly with a capacity error)
    cap = compress_bound(prec, n, CHUNK_N, BATCH_VALUES)
    if w.get("strong"):
        cap = min(cap, 47 + int(n * esz * 0.25))
    d_arc = torch.empty(cap, dtype=torch.uint8, device=dev)
    d_back = torch.empty(n, dtype=tdt, device=dev)
    d_nb = torch.zeros(1, dtype=torch.int64, device=dev)   # archive length, device-resident

    # ---- correctness gate (synchronous API), before anything is timed ----
    arc_t, nb = codec.compress_device(d_vals, CHUNK_N, BATCH_VALUES, out=d_arc, stream=sh)
    codec.decompress_device(d_arc, nb, out=d_back, stream=sh)
    torch.cuda.synchronize()
    assert torch.equal(d_back.view(idt), d_vals.view(idt)), "round trip mismatch"
    info = read_header(d_arc[:47].cpu().numpy().tobytes())
    ratio = nb / in_bytes
    parity = {"round_trip_bit_exact": True}
    if rank == 0 and not args.no_parity and host_vals is not None:
        # full-size byte parity with the unmodified reference (oracle/_ref compress_pipeline)
        from oracle.oracle import Ref, ref_available
        if ref_available():
            want = Ref().compress_pipeline(host_vals.numpy(), CHUNK_N, BATCH_VALUES, 16, 0)
            got = d_arc[:nb].cpu().numpy().tobytes()
            parity.update({"reference_archive_equal": got == want, "archive_bytes": nb,
                           "sha256_16": hashlib.sha256(got).hexdigest()[:16]})
            assert got == want, "GPU archive differs from the reference's"
            del want, got

    def step(evs=None):
        if evs is not None:
            codec.set_kernel_events(enc=(evs[0], evs[1]), dec=(evs[2], evs[3]))
        codec.compress_device_async(d_vals, d_arc, d_nb, CHUNK_N, BATCH_VALUES, stream=sh)
        if world > 1:
            # the one exchange step of a sharded archive: every rank's byte total, so shard
            # g lands at 47 + sum_{h<g} (bytes_h - 47) when concatenated
            sizes = torch.zeros(world, dtype=torch.int64, device=dev)
            sizes[rank] = d_nb[0]
            dist.all_reduce(sizes)
        codec.decompress_device_chained(d_arc, d_nb, info, d_back, stream=sh)

    graph = None
    if w.get("graph") and world == 1:
        # launch-bound size: the whole round trip is one CUDA graph (memsets, encode +
        # placement, walker, decoder with its programmatic dependent launch)
        s = torch.cuda.Stream(dev)
        s.wait_stream(stream)
        with torch.cuda.stream(s):
            for _ in range(2):
                codec.compress_device_async(d_vals, d_arc, d_nb, CHUNK_N, BATCH_VALUES, stream=s.cuda_stream)
                codec.decompress_device_chained(d_arc, d_nb, info, d_back, stream=s.cuda_stream)
        stream.wait_stream(s)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            cs = torch.cuda.current_stream().cuda_stream
            codec.compress_device_async(d_vals, d_arc, d_nb, CHUNK_N, BATCH_VALUES, stream=cs)
            codec.decompress_device_chained(d_arc, d_nb, info, d_back, stream=cs)
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        graph.replay() if graph else step()
    torch.cuda.synchronize()
    codec.sync(sh)

    kev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.steps)]
    for evs in kev:          # torch creates the CUDA event lazily on first record
        for e in evs:
            e.record(stream)
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    # inputs + archive + output that fit the 126 MB L2 get an L2 flush (a 256 MB write) before
    # every timed step, outside its events; each step is timed on its own and the steps summed
    flush = None
    if 2 * in_bytes + cap < (126 << 20):
        flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
        fev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(args.steps)]
    clocks = ClockSampler(local_rank)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    time.sleep(0.3)
    t0.record(stream)
    for k in range(args.steps):
        if flush is not None:
            flush.fill_(k & 0xff)
            fev[k][0].record(stream)
        if graph:
            graph.replay()
        else:
            step(kev[k])
        if flush is not None:
            fev[k][1].record(stream)
    t1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    time.sleep(0.1)
    clk = clocks.stop()
    codec.sync(sh)   # raises on any device-side error of the timed steps
    assert int(d_nb.item()) == nb, "timed steps produced a different archive length"
    assert torch.equal(d_back.view(idt), d_vals.view(idt)), "timed round trip mismatch"
    elapsed = t0.elapsed_time(t1) / 1e3
    flushed = flush is not None
    if flushed:
        elapsed = sum(a.elapsed_time(b) for a, b in fev) / 1e3
    if graph:
        # kernel split of one step, measured outside the graph with the same calls
        enc_ms, dec_ms = [], []
        for evs in kev[: min(5, len(kev))]:
            if flushed:
                flush.fill_(0)
            step(evs)
        torch.cuda.synchronize()
        kev = kev[: min(5, len(kev))]
    codec.set_kernel_events()
    del flush
    enc_ms = [e[0].elapsed_time(e[1]) for e in kev]
    dec_ms = [e[2].elapsed_time(e[3]) for e in kev]
    if world > 1:
        t = torch.tensor([elapsed], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed = float(t.item())
        tot = torch.tensor([in_bytes, nb], dtype=torch.int64, device=dev)
        dist.all_reduce(tot)
        all_bytes, all_arc = int(tot[0].item()), int(tot[1].item())
    else:
        all_bytes, all_arc = in_bytes, nb
    value = all_bytes * args.steps / elapsed / 1e9

    # ---- e2e through the host-buffer C ABI (H2D / D2H inside the timed region) ----
    e2e = None
    if not args.no_e2e and w["gen"] != "device":
        e2e = host_round_trips(torch, codec, dev, w, host_vals, nb, cap, world, args, options)
    del d_back

    if rank != 0:
        return
    peak, peak_src = hbm_peak()
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
                "frac": algo / dom_t / 1e9 / peak, "traffic": traffic,
                "kernel": "encode_chunks_kernel (+ sampler, placement)" if dom == "encode" else "decode_chunks_kernel",
                "peak_source": peak_src,
                "per_launch_bytes": algo,
                "compress_ms": 1e3 * enc_avg, "decompress_ms": 1e3 * dec_avg,
                "compress_frac": algo / enc_avg / 1e9 / peak, "decompress_frac": algo / dec_avg / 1e9 / peak,
                "note": "compress = the chunk sampler (phase 1) + every encode launch incl. the fused "
                        "placement + the final placement launch; decompress = frame walker + decoder; "
                        "traffic = DRAM bytes of the dominant codec kernel alone (ncu --set full)"}
    cpu = None
    if world == 1 and not args.no_cpu and host_vals is not None:
        sample_n = min(n, args.cpu_max_values)
        sample_n = n if sample_n == n else (sample_n // BATCH_VALUES) * BATCH_VALUES
        kind, cores, times, _ = cpu_round_trip(host_vals.numpy()[:sample_n], 3, 1)
        med = statistics.median(times)
        cpu = {"value": sample_n * esz / med / 1e9, "unit": "GB/s", "cores": cores, "kind": kind,
               "sample": f"{'all' if sample_n == n else 'first'} {sample_n} values of the workload; "
                         f"compress_pipeline + decompress_pipeline round trip, median of 3 after 1 warm-up"}
    nl = our_launches_per_step(n, prec)
    line = {
        "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * elapsed / args.steps, "higher_is_better": True,
        "scaling": "strong" if w.get("strong") else "weak", "vs_baseline": None,
        "dtype": "f64" if prec == F64 else "f32",
        "data": ("synthetic, generated on each GPU (counter-based field, csrc/field.cuh)" if w["gen"] == "device"
                 else f"synthetic ({'reference mt19937_64 generator' if w['gen'] == 'reference' else 'pinned kind'}, "
                      f"seed {SEED}{' + rank' if world > 1 else ''})"),
        "config": {"workload": w["desc"], "values_per_gpu": n, "values_total": all_bytes // esz,
                   "chunk_n": CHUNK_N, "batch_values": BATCH_VALUES,
                   "ratio": all_arc / all_bytes, "archive_bytes_per_gpu": nb,
                   "compress_gbs": world * in_bytes / enc_avg / 1e9,
                   "decompress_gbs": world * in_bytes / dec_avg / 1e9,
                   "l2": f"inputs {in_bytes / 1e9:.3f} GB per GPU "
                         + ("fit the 126 MB L2: L2 flushed (256 MB write) before every timed step, outside "
                            "its CUDA events; steps timed one by one" if flushed else
                            "exceed the 126 MB L2; no flush"),
                   "cuda_graph": bool(graph),
                   "parallelism": (f"dp{world} ({'strong: batch-range shards of one stream' if w.get('strong') else 'weak: per-rank copies'}"
                                   f"; NCCL all_reduce of archive byte totals for shard placement)") if world > 1
                   else "dp1"},
        "parity": parity,
        "roofline": roofline,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": nl * args.steps,
        "clocks": clk,
    }
    print(json.dumps(line), flush=True)


def host_round_trips(torch, codec, dev, w, host_vals, nb, cap, world, args, options):
    """compress_host + decompress_host from pinned (and for cfg4 also pageable) buffers;
    every byte of both directions is checked once before timing."""
    import torch.distributed as dist
    prec = w["prec"]
    n = host_vals.numel()
    esz = host_vals.element_size()
    in_bytes = n * esz
    opt = options(CHUNK_N, BATCH_VALUES, 16, 0)
    h_arc = torch.empty(nb + 64, dtype=torch.uint8, pin_memory=True)   # the archive's own size
    h_back = torch.empty_like(host_vals, pin_memory=True)
    hv, ha, hb = host_vals.numpy(), h_arc.numpy(), h_back.numpy()
    variants = [("pinned", hv, ha, hb)]
    if w.get("host"):
        variants.append(("pageable", hv.copy(), np.empty_like(ha), np.empty_like(hb)))
    out = None
    for name, v, a_buf, b_buf in variants:
        a = codec.compress_host(v, opt, out=a_buf)
        codec.decompress_host(a, prec, opt, out=b_buf)
        assert len(a) == nb and np.array_equal(b_buf.view(np.uint8), v.view(np.uint8)), f"e2e {name} mismatch"
        tc, td = [], []
        for _ in range(args.e2e_steps):
            if world > 1:
                dist.barrier()
            s0 = time.perf_counter()
            a = codec.compress_host(v, opt, out=a_buf)
            s1 = time.perf_counter()
            codec.decompress_host(a, prec, opt, out=b_buf)
            s2 = time.perf_counter()
            tc.append(s1 - s0)
            td.append(s2 - s1)
        t = [statistics.median(tc), statistics.median(td)]
        if world > 1:
            tt = torch.tensor(t, dtype=torch.float64, device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            t = tt.tolist()
        rec = {"value": world * in_bytes / (t[0] + t[1]) / 1e9, "unit": "GB/s",
               "h2d_bytes_per_step": in_bytes + nb, "d2h_bytes_per_step": nb + in_bytes,
               "ms_per_step": 1e3 * (t[0] + t[1]),
               "compress_gbs": world * in_bytes / t[0] / 1e9, "decompress_gbs": world * in_bytes / t[1] / 1e9}
        if out is None:
            out = rec
            out["buffers"] = name
        else:
            out[name] = rec
    # the host link bounds these numbers: pinned copy bandwidth measured on this box and
    # the fraction of the link-bound time achieved (compress: H2D of values || D2H of the
    # archive; decompress: H2D of the archive || D2H of the values)
    h2d, d2h = link_bandwidth(torch, dev, host_vals)
    bc = max(in_bytes / h2d, nb / d2h)
    bd = max(nb / h2d, in_bytes / d2h)
    out.update({"link_h2d_gbs": h2d / 1e9, "link_d2h_gbs": d2h / 1e9,
                "link_frac": (bc + bd) / (out["ms_per_step"] / 1e3),
                "compress_link_frac": bc / (in_bytes / out["compress_gbs"] / 1e9 * world),
                "decompress_link_frac": bd / (in_bytes / out["decompress_gbs"] / 1e9 * world)})
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="cfg2")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--cpu-max-values", type=int, default=600_000_000,
                    help="cpu_baseline sample cap (values); cfg1-3 run in full")
    ap.add_argument("--ref-max-values", type=int, default=600_000_000,
                    help="reference-arm cap (values); cfg1-3 run in full, cfg4/5 on whole batches")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    # test hook: FALCON_BENCH_ONE_GPU=1 puts every rank on GPU 0 and exchanges over gloo, so
    # the multi-rank path (shards, exchange, max-over-ranks timing) runs on a one-GPU box
    one_gpu = os.environ.get("FALCON_BENCH_ONE_GPU") == "1"
    if one_gpu:
        local_rank = 0
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        if one_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
