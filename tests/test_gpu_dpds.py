"""GPU self-test of the exact fast per-value analysis (dpds.cuh) against the CPU oracle.

For every input: the fast exact loop and the literal loop (std::round + IEEE division)
must equal the oracle's dp_ds_calculate verdict (numeric.hpp:108-140) bit for bit, and
certification at any candidate scale A must never contradict it:
  certified   -> alpha_v <= A, not an exception, lane integer = round(v * 10^A)
  exception   -> the oracle says exception
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

CANDIDATES = [0, 1, 2, 3, 4, 6, 9, 13, 17, 22]


def f64_inputs(rng, n):
    parts = [rng.integers(0, 1 << 64, n, dtype=np.uint64).view(np.float64)]
    digits = rng.integers(1, 16, 2 * n)
    d = np.array([int(rng.integers(10 ** (k - 1), 10 ** k)) for k in digits[: n // 4]], dtype=np.float64)
    d = np.concatenate([d, rng.integers(1, 10 ** 15, 2 * n - len(d)).astype(np.float64)])
    d *= np.where(rng.integers(0, 2, len(d)) == 1, -1.0, 1.0)
    k = rng.integers(0, 23, len(d))
    dec = d / (10.0 ** k)
    parts.append(dec)
    # 1..3 ulp perturbations: the gap test may pass while the reconstruction fails
    steps = rng.integers(1, 4, n)
    pert = dec[:n].copy()
    for s in range(1, 4):
        sel = steps >= s
        pert[sel] = np.nextafter(pert[sel], np.where(rng.integers(0, 2, sel.sum()) == 1, np.inf, -np.inf))
    parts.append(pert)
    # decade boundaries
    dec_b = []
    for e in range(-30, 31):
        x = float(f"1e{e}")
        for sign in (1.0, -1.0):
            y = x
            for _ in range(6):
                dec_b.append(sign * y)
                y = np.nextafter(y, np.inf)
            y = x
            for _ in range(6):
                y = np.nextafter(y, -np.inf)
                dec_b.append(sign * y)
    parts.append(np.array(dec_b))
    parts.append(np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 5e-324, 2.2250738585072014e-308,
                           1.7976931348623157e308, 0.49999999999999994, 1 - 2 ** -53, 0.1, 0.3,
                           9.110900773177071, 1.23456789876543e-9, 1e-22, 2.5, -0.0314, 1.02]))
    return np.concatenate(parts)


def f32_inputs(rng, n):
    parts = [rng.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32).view(np.float32)]
    d = rng.integers(1, 10 ** 6, 2 * n).astype(np.float32)
    d *= np.where(rng.integers(0, 2, len(d)) == 1, np.float32(-1), np.float32(1))
    k = rng.integers(0, 11, len(d))
    p = np.array([np.float32(10.0 ** i) for i in range(11)], np.float32)
    dec = (d / p[k]).astype(np.float32)
    parts.append(dec)
    pert = dec[:n].copy()
    pert = np.nextafter(pert, np.where(rng.integers(0, 2, n) == 1, np.float32(np.inf), np.float32(-np.inf)))
    parts.append(pert.astype(np.float32))
    parts.append(np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 1e-45, 3.4028235e38, 2.5, 1.02, 9.1109,
                           9.110901], np.float32))
    return np.concatenate(parts)


def expected_g(v, A, prec):
    if prec == 0:
        s = v * (10.0 ** A)
        return (np.sign(s) * np.floor(np.abs(s) + 0.5)).astype(np.int64)
    p = np.float32(10.0 ** A)
    s = (v * p).astype(np.float32)
    return (np.sign(s) * np.floor(np.abs(s) + np.float32(0.5))).astype(np.int64)


@pytest.mark.parametrize("prec", [0, 1])
def test_fast_analysis_matches_oracle(codec, oracle, prec):
    rng = np.random.default_rng(2024 + prec)
    v = f64_inputs(rng, 400_000) if prec == 0 else f32_inputs(rng, 400_000)
    ref = oracle.dp_alpha_batch(v)
    d = torch.from_numpy(v).cuda()
    cands = CANDIDATES if prec == 0 else [0, 1, 2, 3, 5, 7, 10]
    for A in cands:
        full, lit, cert_raw, g = codec.selftest_dp(d, A)
        assert not np.any(cert_raw < 0), f"A={A}: certify_fast/certify_lean disagree with dp_certify at {v[cert_raw < 0][:5]}"
        cert = cert_raw & 3
        lean = (cert_raw & 4) != 0
        bad = np.nonzero(full != ref)[0]
        assert len(bad) == 0, f"fast loop differs at {v[bad[:5]]}: {full[bad[:5]]} vs {ref[bad[:5]]}"
        bad = np.nonzero(lit != ref)[0]
        assert len(bad) == 0, f"literal loop differs at {v[bad[:5]]}"
        ok = cert == 1
        assert np.all((ref[ok] >= 0) & (ref[ok] <= A)), f"A={A}: certified a value the oracle rejects"
        assert np.all(ref[cert == 2] == -1), f"A={A}: certified exception the oracle accepts"
        with np.errstate(all="ignore"):
            ge = expected_g(v[ok], A, prec)
        assert np.array_equal(g[ok], ge), f"A={A}: certified lane integer differs"
        assert np.all(ok[lean]), f"A={A}: lean certification accepted a value dp_certify does not"


def test_certification_rate_on_clean_decimals(codec):
    # not a parity property: the fast path must actually decide typical data
    from paper_2511_04140_b200 import synth
    v = synth("outlier", 1 << 20, 0, dp=2, seed=5, period=100)
    _, _, cert, _ = codec.selftest_dp(torch.from_numpy(v).cuda(), 2)
    assert ((cert & 3) == 1).mean() > 0.999
    assert ((cert & 4) != 0).mean() > 0.999   # the encoder's lean form decides them too


@pytest.mark.parametrize("prec", [0, 1])
def test_division_free_inverse_scale_is_correctly_rounded(codec, prec):
    """The decoder's Markstein inverse scale (dpds.cuh) equals IEEE g / 10^alpha for every
    alpha it is used at (numeric.hpp:159-162: (T)g / pow10<T>(alpha))."""
    rng = np.random.default_rng(77 + prec)
    top = 63 if prec == 0 else 31
    parts = [rng.integers(-(1 << 53), 1 << 53, 600_000, dtype=np.int64),
             rng.integers(-(1 << 20), 1 << 20, 300_000, dtype=np.int64),
             rng.integers(-(1 << (top - 1)), 1 << (top - 1), 300_000, dtype=np.int64),
             np.arange(-5000, 5000, dtype=np.int64)]
    g = np.concatenate(parts)
    if prec == 1:
        g = g.astype(np.int32).astype(np.int64)   # f32 lanes carry int32 integers
    d = torch.from_numpy(g).cuda()
    for alpha in range(0, 22 if prec == 0 else 10):
        got = codec.selftest_div(d, alpha, prec)
        if prec == 0:
            want = g.astype(np.float64) / np.float64(10.0 ** alpha)
            assert np.array_equal(got.view(np.uint64), want.view(np.uint64)), f"alpha={alpha}"
        else:
            p = np.float32(1)
            for _ in range(alpha):
                p = np.float32(p * np.float32(10))
            want = g.astype(np.float32) / p
            assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), f"alpha={alpha}"
