"""Full-size parity against the unmodified reference (oracle/_ref, the reference's own
compress_pipeline / decompress_pipeline, pipeline.hpp:157-365, 371-467) on BASELINE.json's
single-GPU configs at their full sizes:

  cfg1  1,000,000 f64, 2-dp random walk, seed 1 (synthetic.hpp:36-115)
  cfg2  268,435,456 f64, 2-dp walk with 1 % injected outliers (period 100, 3575 units)
  cfg3  536,870,912 f32, reflecting walk, 1-6 dp drawn per 1025-value block (pinned kind)

For each: the GPU archive equals the reference's byte for byte (compared whole, plus a
digest in the failure message), the reference decodes the GPU archive bit-exactly, and the
GPU decodes it bit-exactly too.
"""
import hashlib

import numpy as np
import pytest
import torch

from paper_2511_04140_b200 import F32, F64, synth

pytestmark = pytest.mark.gpu

CONFIGS = {
    "cfg1": ("walk", F64, 1_000_000, dict(dp=2, seed=1)),
    "cfg2": ("outlier", F64, 268_435_456, dict(dp=2, seed=1, period=100, units=3575)),
    "cfg3": ("mixed", F32, 536_870_912, dict(seed=1, block=1025)),
}


@pytest.mark.parametrize("name", sorted(CONFIGS))
def test_full_size_archive_equals_reference(codec, ref, name):
    kind, prec, n, kw = CONFIGS[name]
    vals = synth(kind, n, prec, step=127, **kw)
    d = torch.from_numpy(vals).cuda()
    arc, nb = codec.compress_device(d)
    got = arc[:nb].cpu().numpy()
    want = np.frombuffer(ref.compress_pipeline(vals), np.uint8)
    dg = hashlib.sha256(got.tobytes()).hexdigest()[:16]
    dw = hashlib.sha256(want.tobytes()).hexdigest()[:16]
    assert len(got) == len(want) and np.array_equal(got, want), \
        f"{name}: GPU archive {len(got)} B sha {dg} != reference {len(want)} B sha {dw}"
    # the reference decodes the GPU archive, the GPU decodes it too, both bit-exact
    back_ref = ref.decompress_pipeline(got.tobytes(), prec)
    assert np.array_equal(back_ref.view(np.uint8), vals.view(np.uint8)), f"{name}: reference decode differs"
    del back_ref
    back = codec.decompress_device(arc, nb)
    iv = torch.int64 if prec == F64 else torch.int32
    assert torch.equal(back.view(iv), d.view(iv)), f"{name}: GPU round trip differs"
