"""CPU: the C-ABI library loads, exports every symbol include/falcon_b200.h declares, and
its host-only entry points agree with the oracle (no GPU calls)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from paper_2511_04140_b200 import falcon as fb

HDR = os.path.join(os.path.dirname(os.path.dirname(__file__)), "include", "falcon_b200.h")


def declared_symbols():
    text = open(HDR).read()
    return sorted(set(re.findall(r"\b(falcon_[a-z0-9_]+)\s*\(", text)) - {"falcon_read_fn"})


def test_library_exports_every_declared_symbol():
    lib = fb.load()
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    assert set(fb.EXPORTED) <= set(declared_symbols())


def test_abi_version():
    assert fb.load().falcon_abi_version() == 1


@pytest.mark.parametrize("prec,n", [(0, 65), (0, 1025), (1, 1025), (0, 4097)])
def test_max_encoded_chunk_size(oracle, prec, n):
    assert fb.max_encoded_chunk_size(prec, n) == oracle.max_chunk(prec, n)


@pytest.mark.parametrize("count,n,bv", [(0, 1025, 4198400), (1_000_000, 1025, 4198400), (5000, 65, 1000)])
def test_compress_bound(oracle, count, n, bv):
    assert fb.compress_bound(0, count, n, bv) == oracle.compress_bound(0, count, n, bv)


def test_header_round_trip(oracle):
    arc = oracle.compress_archive(np.arange(5000, dtype=np.float64) / 100, 1025, 2050)
    info = fb.read_header(arc)
    assert (info.precision, info.chunk_n, info.batch_values, info.total_values, info.batch_count) == (0, 1025, 2050, 5000, 3)
    out = (C.c_uint8 * 47)()
    fb.load().falcon_write_header(C.byref(info), out)
    assert bytes(out) == arc[:47]
    with pytest.raises(fb.CorruptError, match="bad archive magic"):
        fb.read_header(b"Y" + arc[1:47])


@pytest.mark.parametrize("kind", ["walk", "decimal", "signflip", "outlier", "bits", "mixed"])
@pytest.mark.parametrize("prec", [0, 1])
def test_synthetic_inputs_match_oracle(oracle, kind, prec):
    a = fb.synth(kind, 30000, prec, seed=5, period=100)
    b = oracle.synth(kind, 30000, prec, seed=5, period=100)
    assert a.view(np.uint8).tobytes() == b.view(np.uint8).tobytes()


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(fb.FalconError):
        fb.Codec(0)
