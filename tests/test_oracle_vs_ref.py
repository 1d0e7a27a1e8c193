"""CPU: the C restatement against the unmodified reference library (oracle/_ref),
on random inputs of every generator kind, both precisions and several geometries."""
import numpy as np
import pytest

from oracle.oracle import F32, F64, OracleError, RefError

KINDS = ["walk", "decimal", "signflip", "outlier", "bits"]


@pytest.mark.parametrize("prec", [F64, F32])
@pytest.mark.parametrize("kind", KINDS)
def test_generators_identical(oracle, ref, kind, prec):
    a = oracle.synth(kind, 20000, prec, seed=11, period=100)
    b = ref.synth(kind, 20000, prec, seed=11, period=100)
    assert a.view(np.uint8).tobytes() == b.view(np.uint8).tobytes()


@pytest.mark.parametrize("prec", [F64, F32])
@pytest.mark.parametrize("kind", KINDS)
def test_chunks_and_archives_match_reference(oracle, ref, kind, prec):
    vals = ref.synth(kind, 30000, prec, seed=21, period=100)
    for n in (65, 257, 1025):
        for i in range(0, 30000 - n, 6007):
            c = vals[i:i + n]
            assert oracle.compress_chunk(c) == ref.compress_chunk(c)
    for n, bv in ((65, 1000), (1025, 4100), (257, 257 * 5)):
        assert oracle.compress_archive(vals, n, bv) == ref.compress_pipeline(vals, n, bv)


def test_dp_ds_matches_reference_on_random_inputs(oracle, ref):
    rng = np.random.default_rng(3)
    vals = np.concatenate([rng.integers(0, 1 << 64, 3000, dtype=np.uint64).view(np.float64),
                           rng.integers(-10 ** 9, 10 ** 9, 3000) / 10.0 ** rng.integers(0, 23, 3000)])
    for v in vals:
        assert oracle.dp_ds(float(v)) == ref.dp_ds(float(v))


def test_corruption_messages_match_reference(oracle, ref):
    vals = ref.synth("walk", 3 * 1025 * 2 + 100, F64, seed=9)
    arc = ref.compress_pipeline(vals, 1025, 1025 * 2)
    rng = np.random.default_rng(1)
    for trial in range(60):
        a = bytearray(arc)
        if trial % 3 == 0:
            a = a[: rng.integers(47, len(a))]
        else:
            pos = int(rng.integers(47, len(a)))
            a[pos] ^= int(rng.integers(1, 256))
        a = bytes(a)
        try:
            ref.decompress_pipeline(a, F64)
            ref_msg = None
        except RefError as e:
            ref_msg = e.message
        try:
            oracle.decompress_archive(a, F64)
            or_msg = None
        except OracleError as e:
            or_msg = e.message
        assert or_msg == ref_msg
