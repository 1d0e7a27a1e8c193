"""GPU: the product reproduces every archive the unmodified reference produced
(tests/golden, made by tests/golden/make_golden.py) and decodes it back bit-exactly,
through the device-resident and the host-pipeline entry points."""
import json
import os

import numpy as np
import pytest
import torch

from paper_2511_04140_b200 import options

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
MAN = json.load(open(os.path.join(GOLDEN, "manifest.json")))


def load(name):
    m = MAN[name]
    vals = np.fromfile(os.path.join(GOLDEN, name + ".in.bin"), dtype=m["dtype"])
    arc = open(os.path.join(GOLDEN, name + ".fln"), "rb").read()
    return m, vals, arc


@pytest.mark.parametrize("name", sorted(MAN))
def test_device_compress_matches_reference_bytes(codec, name):
    m, vals, arc = load(name)
    d = torch.from_numpy(vals).cuda() if len(vals) else torch.empty(0, dtype=getattr(torch, m["dtype"]), device="cuda")
    out, nb = codec.compress_device(d, m["chunk_n"], m["batch_values"])
    assert out[:nb].cpu().numpy().tobytes() == arc
    back = codec.decompress_device(torch.frombuffer(bytearray(arc), dtype=torch.uint8).cuda(), len(arc))
    assert back.cpu().numpy().view(np.uint8).tobytes() == vals.view(np.uint8).tobytes()


@pytest.mark.parametrize("name", sorted(MAN))
def test_host_pipeline_matches_reference_bytes(codec, name):
    m, vals, arc = load(name)
    prec = 0 if m["dtype"] == "float64" else 1
    opt = options(m["chunk_n"], m["batch_values"], 4, 2)
    assert codec.compress_host(vals, opt).tobytes() == arc
    back = codec.decompress_host(arc, prec, opt)
    assert back.view(np.uint8).tobytes() == vals.view(np.uint8).tobytes()
