"""The `falcon` CLI (tools/falcon_cli.cpp): same subcommands and key=value report as the
reference tool (proj/tools/falcon_cli.cpp:251-512).  CPU part: inspect / gen, which need
no GPU; GPU part: compress -> inspect -> verify -> decompress round trips whose archives
must equal the CPU oracle's byte for byte."""
import json
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "tools", "bin", "falcon")
GOLD = os.path.join(ROOT, "tests", "golden")


@pytest.fixture(scope="module")
def cli():
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tools")], check=True)
    return CLI


def run(cli, *args, ok=True):
    r = subprocess.run([cli, *map(str, args)], capture_output=True, text=True)
    if ok:
        assert r.returncode == 0, r.stderr
    return r.returncode, dict(line.split("=", 1) for line in r.stdout.splitlines() if "=" in line), r.stderr


def test_inspect_matches_fixture_headers(cli):
    man = json.load(open(os.path.join(GOLD, "manifest.json")))
    for name, m in man.items():
        _, rep, _ = run(cli, "inspect", os.path.join(GOLD, name + ".fln"))
        assert int(rep["archive_bytes"]) == m["archive_bytes"]
        assert int(rep["chunk_n"]) == m["chunk_n"]
        assert int(rep["batch_values"]) == m["batch_values"]
        assert int(rep["total_values"]) == m["count"]
        assert rep["precision"] == ("64" if m["dtype"] == "float64" else "32")


def test_inspect_rejects_trailing_bytes(cli, tmp_path):
    data = open(os.path.join(GOLD, "outlier_f64_p100.fln"), "rb").read()
    bad = tmp_path / "bad.fln"
    bad.write_bytes(data + b"\0")
    rc, _, err = run(cli, "inspect", bad, ok=False)
    assert rc == 1 and "trailing bytes after final batch" in err   # pipeline.hpp:461


@pytest.mark.parametrize("kind,prec", [("walk", 64), ("outlier", 64), ("decimal", 32), ("bits", 32)])
def test_gen_matches_reference_generator(cli, oracle, tmp_path, kind, prec):
    out = tmp_path / "v.raw"
    _, rep, _ = run(cli, "gen", out, "--kind", kind, "--count", 5000, "--precision", prec, "--seed", 9)
    assert rep == {"values": "5000", "kind": kind}
    got = np.fromfile(out, np.float64 if prec == 64 else np.float32)
    from paper_2511_04140_b200 import synth
    want = synth(kind, 5000, 0 if prec == 64 else 1, dp=2, seed=9, period=1025)
    assert got.tobytes() == want.tobytes()


@pytest.mark.gpu
@pytest.mark.parametrize("prec", [64, 32])
def test_round_trip_through_the_cli(cli, oracle, tmp_path, prec):
    raw, fln, back = tmp_path / "v.raw", tmp_path / "v.fln", tmp_path / "back.raw"
    run(cli, "gen", raw, "--kind", "outlier", "--count", 123457, "--precision", prec, "--period", 100)
    _, rep, _ = run(cli, "compress", raw, fln, "--precision", prec, "--batch-values", 50000, "--streams", 3)
    vals = np.fromfile(raw, np.float64 if prec == 64 else np.float32)
    want = oracle.compress_archive(vals, 1025, 50000)
    assert open(fln, "rb").read() == want
    assert int(rep["values"]) == len(vals) and int(rep["archive_bytes"]) == len(want)
    assert int(rep["batches"]) == 3
    _, ins, _ = run(cli, "inspect", fln)
    assert int(ins["total_values"]) == len(vals) and int(ins["batch_count"]) == 3
    _, ver, _ = run(cli, "verify", raw, fln, "--streams", 2)
    assert ver["verify"] == "ok"
    run(cli, "decompress", fln, back)
    assert open(back, "rb").read() == open(raw, "rb").read()
    # a corrupted original is reported as a mismatch with the first index
    corrupt = bytearray(open(raw, "rb").read())
    corrupt[8 * 777 if prec == 64 else 4 * 777] ^= 1
    (tmp_path / "c.raw").write_bytes(bytes(corrupt))
    rc, ver, _ = run(cli, "verify", tmp_path / "c.raw", fln, ok=False)
    assert rc == 1 and ver["verify"] == "mismatch" and ver["detail"] == "value mismatch at index 777"


@pytest.mark.gpu
def test_csv_round_trip_and_device_bench(cli, tmp_path):
    csv, fln, back = tmp_path / "v.csv", tmp_path / "v.fln", tmp_path / "back.csv"
    run(cli, "gen", csv, "--kind", "walk", "--count", 20000, "--format", "csv")
    run(cli, "compress", csv, fln, "--format", "csv")
    _, ver, _ = run(cli, "verify", csv, fln, "--format", "csv")
    assert ver["verify"] == "ok"
    run(cli, "decompress", fln, back, "--format", "csv")
    assert open(back).read() == open(csv).read()
    _, rep, _ = run(cli, "bench", "--kind", "outlier", "--count", 2000000, "--period", 100, "--device", "--reps", 3)
    assert rep["mode"] == "device" and float(rep["ratio"]) < 0.2
