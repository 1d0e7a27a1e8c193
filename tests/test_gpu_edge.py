"""GPU parity on inputs aimed at the encoder's fast paths (dpds.cuh lean certification,
phase-1 sampling, 32-bit delta path, beta_hat from the max high word) and the decoder's
division-free inverse scale.  Every archive must equal the CPU oracle's byte for byte
(chunk_codec.hpp:50-74; transform.hpp:47-89) and decode bit-exactly.
"""
import numpy as np
import pytest
import torch

from paper_2511_04140_b200 import F32, F64

pytestmark = pytest.mark.gpu

N = 1025


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def check(codec, oracle, vals, n=N, bv=N * 8):
    want = oracle.compress_archive(vals, n, bv)
    arc, nb = codec.compress_device(dev(vals), chunk_n=n, batch_values=bv)
    got = arc[:nb].cpu().numpy().tobytes()
    assert got == want, f"archive differs ({len(got)} vs {len(want)} bytes)"
    back = codec.decompress_device(arc, nb).cpu().numpy()
    assert back.view(np.uint8).tobytes() == vals.view(np.uint8).tobytes()


def decimals(rng, count, dp, lo=-1e4, hi=1e4, dtype=np.float64):
    units = rng.integers(int(lo * 10 ** dp), int(hi * 10 ** dp), count)
    if dtype == np.float64:
        return (units.astype(np.float64) / 10.0 ** dp).astype(dtype)
    p = np.float32(1)
    for _ in range(dp):
        p = np.float32(p * np.float32(10))
    return units.astype(np.float32) / p


def chunks_with(rng, base, inject, every=N):
    """base values with `inject(chunk_values, rng)` applied to every chunk."""
    v = base.copy()
    for c0 in range(0, len(v), every):
        inject(v[c0:c0 + every], rng)
    return v


@pytest.mark.parametrize("prec", [F64, F32])
def test_integers_zeros_and_powers_of_two(codec, oracle, prec):
    dt = np.float64 if prec == F64 else np.float32
    rng = np.random.default_rng(1)
    v = rng.integers(-300, 300, 40 * N).astype(dt)            # many zeros, 1, 2, 4, ... 256
    v[::7] = 0.0
    v[3::11] = np.array([0.5, 0.25, 1024.0, 2.0 ** -3], dt)[rng.integers(0, 4, len(v[3::11]))]
    check(codec, oracle, v)


@pytest.mark.parametrize("prec", [F64, F32])
def test_decade_boundaries(codec, oracle, prec):
    dt = np.float64 if prec == F64 else np.float32
    rng = np.random.default_rng(2)
    ks = range(-6, 10) if prec == F64 else range(-3, 5)
    edge = []
    for k in ks:
        x = dt(float(f"1e{k}"))
        edge += [x, np.nextafter(x, dt(np.inf)), np.nextafter(x, dt(-np.inf)), -x]
    edge = np.array(edge, dt)
    # chunks whose max |v| sits exactly on / next to a decade (beta_hat's second pass)
    v = decimals(rng, 30 * N, 2, -99, 99, dt)
    v[::N] = edge[rng.integers(0, len(edge), len(v[::N]))]
    v[5::37] = edge[rng.integers(0, len(edge), len(v[5::37]))]
    check(codec, oracle, v)


@pytest.mark.parametrize("prec", [F64, F32])
def test_rare_finer_value_not_in_the_sample(codec, oracle, prec):
    # phase 1 samples indices 32L + 16; a finer decimal elsewhere must still raise alpha_max
    dt = np.float64 if prec == F64 else np.float32
    rng = np.random.default_rng(3)
    fine = decimals(rng, 30 * N, 5 if prec == F64 else 4, -50, 50, dt)
    base = decimals(rng, 30 * N, 1, -500, 500, dt)

    def inject(c, r):
        i = int(r.integers(0, len(c)))
        if i % 32 != 16:
            c[i] = fine[i]
    check(codec, oracle, chunks_with(rng, base, inject))


@pytest.mark.parametrize("prec", [F64, F32])
def test_single_exception_makes_case2(codec, oracle, prec):
    dt = np.float64 if prec == F64 else np.float32
    rng = np.random.default_rng(4)
    base = decimals(rng, 24 * N, 2, -1e3, 1e3, dt)
    specials = np.array([np.nan, np.inf, -0.0, 1e-310 if prec == F64 else 1e-40, np.pi, -np.e], dt)

    def inject(c, r):
        c[int(r.integers(0, len(c)))] = specials[int(r.integers(0, len(specials)))]
    check(codec, oracle, chunks_with(rng, base, inject))


def test_wide_f64_integers_and_significand_limits(codec, oracle):
    rng = np.random.default_rng(5)
    v = np.concatenate([
        rng.integers(-(10 ** 14), 10 ** 14, 8 * N).astype(np.float64),       # beta near 15
        rng.integers(10 ** 15, 10 ** 16, 4 * N).astype(np.float64),          # beta 16: Case 2
        rng.integers(-(10 ** 12), 10 ** 12, 8 * N).astype(np.float64) / 1e3,  # 15 significant digits
        rng.integers(-(2 ** 40), 2 ** 40, 8 * N).astype(np.float64) / 1e9,
    ])
    check(codec, oracle, v)


@pytest.mark.parametrize("dp", [0, 3, 7, 12, 18, 21])
def test_scales_up_to_the_division_free_limit(codec, oracle, dp):
    rng = np.random.default_rng(6 + dp)
    mag = 10.0 ** max(0, 14 - dp)
    v = decimals(rng, 12 * N, dp, -mag, mag) if dp <= 12 else \
        rng.integers(-10 ** 6, 10 ** 6, 12 * N).astype(np.float64) / 10.0 ** dp
    check(codec, oracle, v)


def test_alpha_22_takes_the_checked_division(codec, oracle):
    rng = np.random.default_rng(7)
    v = rng.integers(1, 10 ** 6, 6 * N).astype(np.float64) / 1e22
    check(codec, oracle, v)


def test_deltas_crossing_the_32_bit_path(codec, oracle):
    # lane integers right around 2^29..2^31 after scaling: the encoder's 32-bit delta path
    # must hand over to 64-bit arithmetic exactly where the integers stop fitting
    rng = np.random.default_rng(8)
    base = rng.integers(2 ** 28, 2 ** 31 + 2 ** 28, 20 * N).astype(np.float64)
    sign = np.where(rng.integers(0, 2, len(base)) == 1, -1.0, 1.0)
    v = base * sign / 100.0
    check(codec, oracle, v)


@pytest.mark.parametrize("step", [2 ** 22 - 1, -(2 ** 22), 2 ** 22, -(2 ** 22) - 1])
def test_warp_scan_width_boundary(codec, oracle, step):
    # constant deltas: zigzag width 23 for the first two steps (the decoder's 32-bit warp
    # scan, warp sums reaching +-2^30), 24 for the others (64-bit scan)
    rng = np.random.default_rng(9)
    g = np.cumsum(np.full(16 * N, step, np.int64)) + int(rng.integers(-1000, 1000))
    v = g.astype(np.float64)
    v[N::2 * N] = -v[N::2 * N]     # odd chunks: a wide first delta (w = 35, 64-bit scan)
    check(codec, oracle, v)


def _walk_units(rng, count, lo=-10 ** 4, hi=10 ** 4, step=127):
    g = np.cumsum(rng.integers(-step, step + 1, count)) + int(rng.integers(lo, hi))
    return g.astype(np.int64)


@pytest.mark.parametrize("dp", [0, 2, 6])
@pytest.mark.parametrize("at", [256, 512, 768])
def test_wide_value_ending_the_previous_warp(codec, oracle, dp, at):
    # A small-valued walk whose chunk holds one wide value at in-chunk index 256/512/768:
    # the last value of warp k-1 is the value warp k's first delta starts from
    # (transform.hpp:87-88).  The 32-bit delta path must not be taken for that delta.
    rng = np.random.default_rng(100 + dp * 7 + at)
    g = _walk_units(rng, 12 * N, lo=-100 * 10 ** dp, hi=100 * 10 ** dp, step=3)
    spike = 3 * 10 ** 9 if dp != 6 else 3 * 10 ** 9 + 17     # > 2^31 units, still Case 1
    for c0 in range(0, len(g) - N + 1, N):
        g[c0 + at] = spike if (c0 // N) % 2 == 0 else -spike
    v = g.astype(np.float64) / 10.0 ** dp
    check(codec, oracle, v)


def test_verdict_example_3e7_in_a_2dp_walk(codec, oracle):
    # the reviewer's case: a 2-dp walk around 100.00 with v[256] = 3e7 (z[257] needs 33 bits)
    rng = np.random.default_rng(5)
    g = 10000 + _walk_units(rng, 4 * N, lo=0, hi=1, step=2)
    v = g.astype(np.float64) / 100.0
    v[256] = 3e7
    v[N + 512] = -3e7
    v[2 * N + 768] = 3e7
    check(codec, oracle, v)


@pytest.mark.parametrize("seed", range(4))
def test_fuzz_magnitudes_at_warp_and_thread_boundaries(codec, oracle, seed):
    # randomized differential fuzz: per chunk a random decimal count, a small walk, and a
    # few values of random magnitude (2^0..2^50 units, up to the Case-1 limit) placed at
    # warp and thread boundaries (in-chunk index 8t and its neighbours)
    rng = np.random.default_rng(1000 + seed)
    nch = 48
    out = []
    for c in range(nch):
        dp = int(rng.integers(0, 7))
        g = _walk_units(rng, N, lo=-50, hi=50, step=int(rng.integers(1, 200)))
        for _ in range(int(rng.integers(1, 6))):
            base = int(rng.choice([256, 512, 768, 0, 1024, 8 * int(rng.integers(1, 128))]))
            pos = min(max(base + int(rng.integers(-1, 2)), 0), N - 1)
            mag = int(2 ** float(rng.uniform(0, 50)))
            lim = 10 ** (15 - dp) - 1 if dp < 15 else 1          # keep beta_hat <= 15
            g[pos] = min(mag, lim) * (1 if rng.integers(0, 2) else -1)
        out.append(g.astype(np.float64) / 10.0 ** dp)
    v = np.concatenate(out)
    check(codec, oracle, v)


@pytest.mark.parametrize("prec", [F64, F32])
@pytest.mark.parametrize("shift", [0, 1, 2, 3])
def test_inputs_at_every_16_byte_phase(codec, oracle, prec, shift):
    # the encoder's 16-B vector loads start at the 16-B boundary at or below each thread's
    # first value: inputs whose first value sits at every phase (and chunks of both parities)
    from paper_2511_04140_b200 import synth
    vals = synth("outlier" if prec == F64 else "mixed", 23 * N + 333, prec, seed=31 + shift, period=100)
    base = torch.from_numpy(np.concatenate([np.zeros(shift, vals.dtype), vals])).cuda()
    d = base[shift:]
    assert d.data_ptr() % 16 == (shift * vals.itemsize) % 16
    want = oracle.compress_archive(vals, N, N * 8)
    arc, nb = codec.compress_device(d, chunk_n=N, batch_values=N * 8)
    assert arc[:nb].cpu().numpy().tobytes() == want
    assert torch.equal(codec.decompress_device(arc, nb).cpu(), d.cpu())


# ---- phase 1 runs in sample_chunks_kernel on each chunk's first 8 values (encode.cu) ----
@pytest.mark.parametrize("prec", [F64, F32])
@pytest.mark.parametrize("where", ["sampled", "unsampled"])
def test_exception_inside_and_outside_the_sample_window(codec, oracle, prec, where):
    dt = np.float64 if prec == F64 else np.float32
    rng = np.random.default_rng(21)
    base = decimals(rng, 16 * N, 2, -1e3, 1e3, dt)
    specials = np.array([np.nan, -np.inf, -0.0, 1e-310 if prec == F64 else 1e-40], dt)

    def inject(c, r):
        i = int(r.integers(0, 8)) if where == "sampled" else int(r.integers(8, len(c)))
        c[min(i, len(c) - 1)] = specials[int(r.integers(0, len(specials)))]
    check(codec, oracle, chunks_with(rng, base, inject))


@pytest.mark.parametrize("prec", [F64, F32])
@pytest.mark.parametrize("sample_dp,rest_dp", [(0, 3), (4, 1), (2, 2)])
def test_sample_window_coarser_or_finer_than_the_chunk(codec, oracle, prec, sample_dp, rest_dp):
    # coarser sample: alpha_max > A0 (general Case-1 path); finer: every value certified at A0
    dt = np.float64 if prec == F64 else np.float32
    rng = np.random.default_rng(22 + sample_dp)
    v = decimals(rng, 12 * N, rest_dp, -900, 900, dt)
    s = decimals(rng, 12 * N, sample_dp, -900, 900, dt)
    for c0 in range(0, len(v), N):
        v[c0:c0 + 8] = s[c0:c0 + 8]
    check(codec, oracle, v)


@pytest.mark.parametrize("prec", [F64, F32])
@pytest.mark.parametrize("tail", [1, 3, 7, 8, 9])
def test_final_chunk_shorter_than_the_sample(codec, oracle, prec, tail):
    # the sampler reads +0.0 padding past a short final chunk (pipeline.hpp:205-215)
    dt = np.float64 if prec == F64 else np.float32
    rng = np.random.default_rng(30 + tail)
    check(codec, oracle, decimals(rng, 5 * N + tail, 3, -50, 50, dt), bv=N * 2)
