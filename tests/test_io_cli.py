"""FCTN containers and the `complete` / `metrics` CLI.

CPU: the container reader/writer against files the REAL reference wrote
(tests/golden/io, made by tests/golden/make_io_golden.py) — same values, and
byte-identical files when we write the same arrays; the reference's error
cases; CLI usage errors exit 1.  GPU: `metrics` reproduces the reference
CLI's CSV; `complete` writes the oracle's result (FP64 bound 1e-9) and the
reference's report schema."""
import contextlib
import csv
import io
import os
import struct

import numpy as np
import pytest

from paper_2510_22506_b200 import fileio
from paper_2510_22506_b200.cli import main

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "io")


def _arrays():
    rng = np.random.default_rng(7)
    truth = rng.uniform(0, 1, (9, 7, 4))
    est = truth + 0.05 * rng.standard_normal(truth.shape)
    return truth, est


def test_reads_reference_containers():
    truth, est = _arrays()
    assert np.array_equal(fileio.read_tensor(os.path.join(GOLD, "truth.fctn")), truth)
    assert np.array_equal(fileio.read_tensor(os.path.join(GOLD, "est.fctn")), est)
    assert np.array_equal(fileio.read_tensor(os.path.join(GOLD, "vec.fctn")), np.arange(5.0))
    m = fileio.read_mask(os.path.join(GOLD, "mask.fctn"))
    assert m.dtype == bool and np.array_equal(m, fileio.sample_mask(truth.shape, 0.3, 11))  # exact-count sampler


def test_writes_byte_identical_containers(tmp_path):
    truth, est = _arrays()
    for name, arr in [("truth.fctn", truth), ("est.fctn", est), ("vec.fctn", np.arange(5.0))]:
        p = tmp_path / name
        fileio.write_tensor(str(p), arr)
        assert p.read_bytes() == open(os.path.join(GOLD, name), "rb").read(), name
    p = tmp_path / "mask.fctn"
    fileio.write_mask(str(p), fileio.sample_mask(truth.shape, 0.3, 11))
    assert p.read_bytes() == open(os.path.join(GOLD, "mask.fctn"), "rb").read()
    assert not [f for f in os.listdir(tmp_path) if f.startswith(".fctn-")]  # atomic writes leave no temp files


def test_container_errors(tmp_path):
    good = open(os.path.join(GOLD, "truth.fctn"), "rb").read()
    cases = {
        "magic": b"XXXX" + good[4:],
        "version": good[:4] + struct.pack("<I", 2) + good[8:],
        "trunc_header": good[:10],
        "trunc_extents": good[:20],
        "payload": good[:-8],
        "zero_extent": good[:16] + struct.pack("<Q", 0) + good[24:],
    }
    for name, blob in cases.items():
        p = tmp_path / f"{name}.fctn"
        p.write_bytes(blob)
        with pytest.raises(ValueError):
            fileio.read_tensor(str(p))
    with pytest.raises(ValueError):  # element code: a mask read as a tensor and vice versa
        fileio.read_tensor(os.path.join(GOLD, "mask.fctn"))
    with pytest.raises(ValueError):
        fileio.read_mask(os.path.join(GOLD, "truth.fctn"))
    m = bytearray(open(os.path.join(GOLD, "mask.fctn"), "rb").read())
    m[-1] = 2
    p = tmp_path / "badmask.fctn"
    p.write_bytes(bytes(m))
    with pytest.raises(ValueError, match="strictly 0 or 1"):
        fileio.read_mask(str(p))
    with pytest.raises(ValueError):
        fileio.sample_mask((4, 4), 0.0, 0)


def test_cli_usage_errors_exit_1(tmp_path, capsys):
    assert pytest.raises(SystemExit, main, ["complete"]).value.code == 1  # argparse usage -> 1, not 2
    src = os.path.join(GOLD, "truth.fctn")
    out = str(tmp_path / "x.fctn")
    assert main(["complete", "--input", src, "--output", out]) == 1  # neither --mask nor --sr
    assert main(["complete", "--input", src, "--output", out, "--sr", "0.5",
                 "--mask", os.path.join(GOLD, "mask.fctn")]) == 1
    assert main(["complete", "--input", src, "--output", out, "--sr", "0.5", "--max-rank", "1,2"]) == 1
    assert main(["metrics", "--truth", src, "--est", os.path.join(GOLD, "vec.fctn")]) == 1  # shape mismatch
    assert main(["complete", "--input", str(tmp_path / "missing.fctn"), "--output", out, "--sr", "0.5"]) == 1
    assert not os.path.exists(out)


@pytest.mark.gpu
def test_gpu_cli_metrics_matches_reference_cli(capsys):
    rc = main(["metrics", "--truth", os.path.join(GOLD, "truth.fctn"), "--est", os.path.join(GOLD, "est.fctn"),
               "--mask", os.path.join(GOLD, "mask.fctn")])
    assert rc == 0
    got = list(csv.reader(io.StringIO(capsys.readouterr().out)))
    want = list(csv.reader(open(os.path.join(GOLD, "metrics.csv"))))
    assert got[0] == want[0] == ["psnr", "ssim", "rel_err", "rel_err_offmask"]
    for g, w in zip(got[1], want[1]):
        assert float(g) == pytest.approx(float(w), rel=1e-9)
    assert main(["metrics", "--truth", os.path.join(GOLD, "truth.fctn"),
                 "--est", os.path.join(GOLD, "est.fctn")]) == 0
    row = list(csv.reader(io.StringIO(capsys.readouterr().out)))[1]
    assert row[3] == "nan"


@pytest.mark.gpu
@pytest.mark.parametrize("alg", ["fctnlr", "afctnlr"])
def test_gpu_cli_complete_matches_oracle(tmp_path, alg):
    from oracle import fctn_oracle as O
    truth, _ = _arrays()
    src = str(tmp_path / "obs.fctn")
    fileio.write_tensor(src, truth)
    out, rep, mpath = str(tmp_path / "x.fctn"), str(tmp_path / "rep.csv"), str(tmp_path / "m.fctn")
    buf = io.StringIO()
    with contextlib.redirect_stdout(buf):
        rc = main(["complete", "--input", src, "--output", out, "--sr", "0.4", "--seed", "3", "--save-mask", mpath,
                   "--report", rep, "--algorithm", alg, "--max-rank", "2", "--max-iters", "12", "--eps", "0",
                   "--rank-policy", "fixed", "--initial-rank", "2"])
    assert rc == 0 and buf.getvalue().startswith("completed: iterations=12")
    mask = fileio.read_mask(mpath)
    assert np.array_equal(mask, fileio.sample_mask(truth.shape, 0.4, 3))
    ref = O.run(np.where(mask, truth, 0.0), mask, lam=0.35, delta=0.5, rho=0.1, eps=0.0, max_iters=12, max_rank=2,
                initial_rank=2, rank_policy="fixed", algorithm=alg, shuffle=True, seed=3)
    x = fileio.read_tensor(out)
    assert np.linalg.norm(x - ref.x) <= 1e-9 * np.linalg.norm(ref.x)
    rows = list(csv.DictReader(open(rep)))
    assert list(rows[0].keys()) == ["iteration", "objective", "rel_change", "wall_ms", "flops", "cache_hits", "rank"]
    assert [int(r["flops"]) for r in rows] == [t.flops for t in ref.trace]
    assert rows[0]["rank"] == "2|2|2"
