"""Generate the golden fixtures under tests/golden/ from the UNMODIFIED reference library.

Run in the build container (needs /root/reference, built into oracle/_ref by
`make -C oracle ref`):   python tests/golden/make_golden.py

Each fixture is <name>.in.bin (raw little-endian values), <name>.fln (the archive the
reference's compress_pipeline produced) and an entry in manifest.json with the
geometry.  The GPU tests compare the product against these bytes; the CPU tests pin
the C restatement (oracle/) against them.  Inputs come from the reference generators
(synthetic.hpp:36-115) plus the reference tests' special-value list
(acceptance.cpp:42-77).
"""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.oracle import F32, F64, Ref  # noqa: E402

SPECIALS_F64 = np.array([0.0, -0.0, np.inf, -np.inf, np.nan,
                         np.frombuffer(np.uint64(0x7ff4000000000001).tobytes(), np.float64)[0],
                         np.frombuffer(np.uint64(0xfff8000000000123).tobytes(), np.float64)[0],
                         5e-324, -5e-324, 4.9e-324, 1.7976931348623157e308, -1.7976931348623157e308,
                         2.2250738585072014e-308, 1.0, -1.0])
SPECIALS_F32 = np.array([0.0, -0.0, np.inf, -np.inf, np.nan,
                         np.frombuffer(np.uint32(0x7fa00001).tobytes(), np.float32)[0],
                         np.frombuffer(np.uint32(0xffc00123).tobytes(), np.float32)[0],
                         1e-45, -1e-45, 3.4028235e38, -3.4028235e38, 1.1754944e-38, 1.0, -1.0], np.float32)


def cases(ref: Ref):
    out = []
    # cfg1 shape: reference generator, random walk, 2 dp, seed 1 (first 100k values)
    out.append(("walk_f64_dp2_seed1", ref.synth("walk", 100_000, F64, dp=2, seed=1), 1025, 1025 * 1024 * 4))
    out.append(("outlier_f64_p100", ref.synth("outlier", 60_000, F64, dp=2, seed=3, period=100), 1025, 1025 * 16))
    out.append(("decimal_f64_dp3", ref.synth("decimal", 20_000, F64, dp=3, seed=4), 257, 5000))
    out.append(("signflip_f64", ref.synth("signflip", 8_000, F64, seed=5), 65, 1000))
    out.append(("bits_f64", ref.synth("bits", 6_000, F64, seed=6), 1025, 4100))
    seasoned = np.concatenate([SPECIALS_F64, ref.synth("walk", 5_000, F64, dp=2, seed=7)])
    out.append(("specials_walk_f64", seasoned, 1025, 2 * 1025))
    out.append(("walk_f32_dp1", ref.synth("walk", 50_000, F32, dp=1, seed=8), 1025, 1025 * 8))
    out.append(("bits_f32", ref.synth("bits", 6_000, F32, seed=9), 257, 3000))
    seasoned32 = np.concatenate([SPECIALS_F32, ref.synth("decimal", 5_000, F32, dp=2, seed=10)])
    out.append(("specials_decimal_f32", seasoned32, 65, 1000))
    out.append(("empty_f64", np.zeros(0), 1025, 1025 * 1024 * 4))
    # the chunk-level golden vectors of test_chunk_codec.cpp:32-70 as one-chunk archives
    spike = np.zeros(65)
    spike[0] = 2.5
    out.append(("spike_n65", spike, 65, 65))
    out.append(("zeros_n1025", np.zeros(1025), 1025, 1025))
    out.append(("const25_n1025", np.full(1025, 2.5), 1025, 1025))
    return out


def main():
    ref = Ref()
    manifest = {}
    for name, vals, n, bv in cases(ref):
        vals = np.ascontiguousarray(vals)
        arc = ref.compress_pipeline(vals, n, bv, 16, 0)
        back = ref.decompress_pipeline(arc, F64 if vals.dtype == np.float64 else F32)
        assert back.view(np.uint8).tobytes() == vals.view(np.uint8).tobytes(), name
        with open(os.path.join(HERE, name + ".in.bin"), "wb") as f:
            f.write(vals.tobytes())
        with open(os.path.join(HERE, name + ".fln"), "wb") as f:
            f.write(arc)
        manifest[name] = {"dtype": str(vals.dtype), "count": int(len(vals)), "chunk_n": n,
                          "batch_values": bv, "archive_bytes": len(arc),
                          "sha256": hashlib.sha256(arc).hexdigest()}
        print(f"{name:24s} {len(vals):7d} values -> {len(arc):8d} bytes")
    with open(os.path.join(HERE, "manifest.json"), "w") as f:
        json.dump(manifest, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
