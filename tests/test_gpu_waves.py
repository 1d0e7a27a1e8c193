"""Launch shapes that the default sizes do not reach on small inputs, each in its own process
(the knobs are read once per process): several encode waves with the placement of earlier
waves fused into later launches and a wrapping image ring (FALCON_ENC_WAVE_CHUNKS), both
final-placement shapes (FALCON_PLACE_WIDE_BELOW: 0 = always the NT-thread shape, huge =
always the wide one), and the one-role frame walker (FALCON_WALK_SERIAL, the default before
the two-role walk).  Every archive must equal the oracle's byte for byte, every decode the
input bit for bit."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu

CHILD = r"""
import sys
sys.path.insert(0, {root!r})
import numpy as np, torch
from oracle.oracle import Oracle
from paper_2511_04140_b200 import F32, F64, Codec, synth
orc, codec = Oracle(), Codec(0)
for kind, prec, n, bv in (("outlier", F64, 301 * 4 * 1025 + 77, 4 * 1025), ("mixed", F32, 171 * 1025 * 3 + 5, 3 * 1025),
                          ("walk", F64, 40_000, 50_000)):
    vals = synth(kind, n, prec, seed=7, period=100)
    d = torch.from_numpy(vals).cuda()
    arc, nb = codec.compress_device(d, 1025, bv)
    assert arc[:nb].cpu().numpy().tobytes() == orc.compress_archive(vals, 1025, bv), (kind, n)
    back = codec.decompress_device(arc, nb)
    assert torch.equal(back.cpu(), d.cpu())
print("ok")
"""


@pytest.mark.parametrize("env", [
    {"FALCON_ENC_WAVE_CHUNKS": "8"},
    {"FALCON_ENC_WAVE_CHUNKS": "300"},
    {"FALCON_PLACE_WIDE_BELOW": "0"},
    {"FALCON_PLACE_WIDE_BELOW": "1000000000"},
    {"FALCON_WALK_SERIAL": "1"},
])
def test_launch_shapes_match_the_oracle(env):
    r = subprocess.run([sys.executable, "-c", CHILD.format(root=ROOT)], capture_output=True, text=True,
                       timeout=600, env={**os.environ, **env})
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout[-2000:] + r.stderr[-2000:]
