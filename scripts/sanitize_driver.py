"""Small end-to-end exercise of every device kernel for compute-sanitizer runs
(scripts/sanitize.sh): multi-wave encode with fused placement (small wave), walker +
decoder, chained async round trip, batch index + range decode, a corrupt archive, the
host pipeline and the device field generator.  Checked against the oracle."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("FALCON_ENC_WAVE_CHUNKS", "8")     # several waves + ring wrap

from oracle.oracle import Oracle  # noqa: E402
from paper_2511_04140_b200 import (F32, F64, Codec, CorruptError, compress_bound, options,  # noqa: E402
                                   read_header, synth)

orc = Oracle()
codec = Codec(0)
for kind, prec in (("outlier", F64), ("mixed", F32)):
    vals = synth(kind, 45 * 4 * 1025 + 77, prec, seed=3, period=100)
    want = orc.compress_archive(vals, 1025, 4 * 1025)
    d = torch.from_numpy(vals).cuda()
    arc, nb = codec.compress_device(d, 1025, 4 * 1025)
    assert arc[:nb].cpu().numpy().tobytes() == want
    back = codec.decompress_device(arc, nb)
    assert torch.equal(back.cpu(), d.cpu())
    # chained async
    d_nb = torch.zeros(1, dtype=torch.int64, device="cuda")
    out = torch.empty_like(d)
    info = read_header(want[:47])
    codec.compress_device_async(d, arc, d_nb, 1025, 4 * 1025)
    codec.decompress_device_chained(arc, d_nb, info, out)
    codec.sync()
    assert torch.equal(out.cpu(), d.cpu())
    # index + range
    idx = codec.archive_index(arc, nb)
    part = codec.decompress_range(arc, idx, 2, 3).cpu().numpy()
    assert part.tobytes() == vals[2 * 4 * 1025: 5 * 4 * 1025].tobytes()
    # corrupt archive
    bad = bytearray(want)
    bad[len(bad) // 2] ^= 0x5a
    t = torch.frombuffer(bad, dtype=torch.uint8).cuda()
    try:
        codec.decompress_device(t, len(bad))
    except Exception:  # noqa: BLE001
        pass
    # host pipeline
    opt = options(1025, 4 * 1025, 3, 2)
    h = codec.compress_host(vals, opt)
    assert h.tobytes() == want
    assert codec.decompress_host(h, prec, opt).tobytes() == vals.tobytes()
f = torch.empty(50_000, dtype=torch.float64, device="cuda")
codec.synth_device(f, "field", first=12345)
assert f.cpu().numpy().tobytes() == synth("field", 50_000, F64, first=12345).tobytes()
torch.cuda.synchronize()
print("sanitize driver ok")
