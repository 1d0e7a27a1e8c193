#!/usr/bin/env python
"""Copy the judged evidence of one profiling round from gpurun_out/ into profiles/<tag>/:
bench line(s), the ncu launch list, per-kernel ncu summaries (details page, key raw
metrics, stall reasons, per-region instruction shares) and a SUMMARY.md table.
    python scripts/save_profile.py r01_v2 [workload]"""
import csv, io, json, os, shutil, subprocess, sys

tag = sys.argv[1]
W = sys.argv[2] if len(sys.argv) > 2 else "cfg2"
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
src = os.path.join(root, "gpurun_out")
dst = os.path.join(root, "profiles", tag)
os.makedirs(dst, exist_ok=True)

RAW = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread",
       "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
       "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
       "smsp__issue_active.avg.pct_of_peak_sustained_active"]


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


def raw_metrics(rep):
    r = list(csv.reader(io.StringIO(ncu(rep, "--page", "raw", "--csv"))))
    h, u, v = r[0], r[1], r[2]
    out = {}
    for i, name in enumerate(h):
        if name in RAW or ("pcsamp_warps_issue_stalled" in name and not name.endswith("not_issued")):
            out[name] = (v[i], u[i])
    return out


def to_bytes(val, unit):
    x = float(val.replace(",", ""))
    return x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)


for f in [f"bench_full.log", f"bench_{W}.log", "bench_cfg3.log", f"launches_{W}.csv"]:
    p = os.path.join(src, f)
    if os.path.exists(p):
        shutil.copy(p, os.path.join(dst, f))
bench = None
for f in ["bench_full.log", f"bench_{W}.log"]:
    p = os.path.join(src, f)
    if os.path.exists(p):
        bench = json.loads(open(p).read().strip().splitlines()[-1])
        break
rows = []
traffic = {}
for k in ["encode_chunks_kernel", "decode_chunks_kernel", "sample_chunks_kernel"]:
    rep = os.path.join(src, f"prof_{W}_{k}.ncu-rep")
    if not os.path.exists(rep):
        continue
    with open(os.path.join(dst, f"ncu_{k}_details.csv"), "w") as f:
        f.write(ncu(rep, "--page", "details", "--csv"))
    m = raw_metrics(rep)
    with open(os.path.join(dst, f"ncu_{k}_raw.txt"), "w") as f:
        for name, (val, unit) in sorted(m.items()):
            f.write(f"{name} {val} {unit}\n")
    t_ns = float(m["gpu__time_duration.sum"][0].replace(",", "")) * {"ms": 1e6, "us": 1e3, "ns": 1}.get(m["gpu__time_duration.sum"][1], 1)
    rd = to_bytes(*m["dram__bytes_read.sum"])
    wr = to_bytes(*m["dram__bytes_write.sum"])
    traffic[f"{W}_{k.split('_')[0]}"] = rd + wr
    stalls = sorted(((float(v.replace(",", "")), n.replace("smsp__pcsamp_warps_issue_stalled_", ""))
                     for n, (v, _) in m.items() if "pcsamp" in n), reverse=True)[:4]
    rows.append((k, t_ns / 1e6, rd, wr, m.get("smsp__inst_executed.sum", ("?", ""))[0],
                 m.get("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", ("?",))[0],
                 m.get("smsp__issue_active.avg.pct_of_peak_sustained_active", ("?",))[0],
                 ", ".join(s for _, s in stalls)))
with open(os.path.join(root, "profiles", "ncu_traffic.json"), "w") as f:
    json.dump(traffic, f, indent=1)
with open(os.path.join(dst, "SUMMARY.md"), "w") as f:
    f.write(f"# {tag} -- {W}, 1x B200\n\n")
    if bench:
        r = bench["roofline"]
        f.write(f"bench.py (CUDA events, {bench['steps']} steps): value {bench['value']:.1f} GB/s round trip, "
                f"encode kernel {r['encode_kernel_ms']:.3f} ms (frac {r['encode_frac']:.3f}), decode kernel "
                f"{r['decode_kernel_ms']:.3f} ms (frac {r['decode_frac']:.3f}) of {r['peak']} GB/s; ratio "
                f"{bench['config']['ratio']:.4f}.\n\n")
    f.write("| kernel | ncu time (ms) | DRAM read | DRAM write | warp-instr | ALU pipe % | issue active % | top stalls |\n")
    f.write("|---|---|---|---|---|---|---|---|\n")
    for k, t, rd, wr, ins, alu, iss, st in rows:
        f.write(f"| {k} | {t:.3f} | {rd/1e9:.3f} GB | {wr/1e9:.3f} GB | {ins} | {alu} | {iss} | {st} |\n")
print(open(os.path.join(dst, "SUMMARY.md")).read())
