"""CPU: the C restatement (oracle/) pinned to the reference's own golden vectors and
known answers, and to the committed fixtures produced by the unmodified reference."""
import json
import os

import numpy as np
import pytest

from oracle.oracle import F32, F64, OracleError

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def load_fixture(name):
    man = json.load(open(os.path.join(GOLDEN, "manifest.json")))[name]
    vals = np.fromfile(os.path.join(GOLDEN, name + ".in.bin"), dtype=man["dtype"])
    arc = open(os.path.join(GOLDEN, name + ".fln"), "rb").read()
    return man, vals, arc


FIXTURES = sorted(json.load(open(os.path.join(GOLDEN, "manifest.json"))))


@pytest.mark.parametrize("name", FIXTURES)
def test_oracle_reproduces_reference_fixtures(oracle, name):
    man, vals, arc = load_fixture(name)
    assert oracle.compress_archive(vals, man["chunk_n"], man["batch_values"]) == arc
    prec = F64 if man["dtype"] == "float64" else F32
    back = oracle.decompress_archive(arc, prec)
    assert back.view(np.uint8).tobytes() == vals.view(np.uint8).tobytes()


# test_chunk_codec.cpp:32-70, 216-227; FORMAT.md:106-123
def test_chunk_golden_vectors(oracle):
    assert oracle.compress_chunk(np.zeros(1025)) == bytes(11)
    assert oracle.compress_chunk(np.full(1025, 2.5)) == bytes([1, 2, 25] + [0] * 8)
    v = np.zeros(65)
    v[0] = 2.5
    assert oracle.compress_chunk(v).hex() == "010219000000000000000600808080800000008080"
    assert oracle.compress_chunk(np.zeros(1025, np.float32)) == bytes(7)
    assert oracle.compress_chunk(np.full(1025, 2.5, np.float32)) == bytes([1, 2, 25, 0, 0, 0, 0])


# test_numeric.cpp:98-122, 229-243
@pytest.mark.parametrize("v,a,b", [(0.0, 0, 0), (-0.0314, 4, 3), (1.11, 2, 3), (1.02, 2, 3),
                                   (111.0, 0, 3), (2.5, 1, 2), (1e-22, 22, 1)])
def test_dp_ds_known_answers(oracle, v, a, b):
    assert oracle.dp_ds(v)[:2] == (a, b)


@pytest.mark.parametrize("v", [9.110900773177071, 1.23456789876543e-9, -0.0, float("nan"),
                               float("inf"), -float("inf"), 5e-324])
def test_dp_ds_exceptions(oracle, v):
    assert oracle.dp_ds(v)[:2] == (23, 16)


def test_dp_ds_f32(oracle):
    assert oracle.dp_ds(2.5, F32)[:2] == (1, 2)
    assert oracle.dp_ds(np.float32(-0.0314), F32)[:2] == (4, 3)
    assert oracle.dp_ds(np.float32(9.110901), F32)[:2] == (11, 7)
    assert oracle.dp_ds(np.float32(9.1109), F32)[:2] != (11, 7)


# test_numeric.cpp:74-89: exact floor_log10 at decade boundaries
def test_floor_log10_decades(oracle):
    for k in range(-300, 301, 7):
        x = float(f"1e{k}")
        assert oracle.floor_log10(x) == k
        assert oracle.floor_log10(np.nextafter(x, 0)) == k - 1


# test_numeric.cpp:196-207
def test_round_half_away(oracle):
    assert oracle.round_scale(-1.2, 2) == -120
    assert oracle.round_scale(0.25, 1) == 3
    assert oracle.round_scale(-0.25, 1) == -3
    assert oracle.round_scale(8.04, 2) == 804
    assert oracle.round_scale(1e300, 22) is None  # scaled value exceeds 63 bits


# test_chunk_codec.cpp:175-214
def test_chunk_corruption(oracle):
    rng = np.random.default_rng(33)
    vals = (rng.integers(0, 200001, 65) - 100000) / 1000.0
    enc = oracle.compress_chunk(vals)
    for k in range(len(enc)):
        with pytest.raises(OracleError) as e:
            oracle.decompress_chunk(enc[:k], 65, 65)
        assert e.value.corrupt
    with pytest.raises(OracleError, match="chunk size mismatch"):
        oracle.decompress_chunk(enc + b"\0", 65, 65)
    bad = bytearray(enc)
    bad[10] = 65
    with pytest.raises(OracleError, match="plane count out of range"):
        oracle.decompress_chunk(bytes(bad), 65, 65)
    with pytest.raises(OracleError, match="count exceeds chunk capacity"):
        oracle.decompress_chunk(enc, 65, 66)


# test_container.cpp:62-127
def test_container_edges(oracle):
    assert len(oracle.compress_archive(np.zeros(0))) == 47
    arc = oracle.compress_archive(np.zeros(1025), 1025, 1025)
    assert arc[47:55] == bytes([1, 0, 0, 0, 11, 0, 0, 0])
    with pytest.raises(OracleError, match="trailing bytes after final batch"):
        oracle.decompress_archive(arc + b"\0")
    with pytest.raises(OracleError, match="bad archive magic"):
        oracle.decompress_archive(b"X" + arc[1:])
    with pytest.raises(OracleError, match=r"batch payload truncated \(batch 0\)"):
        oracle.decompress_archive(arc[:-1])
