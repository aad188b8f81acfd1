"""Golden container files written by the REAL reference (`fctnlr.fileio`,
fileio.py:59-136).  Run in the authoring container only:

    PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/reference/pkg/src \
        python tests/golden/make_io_golden.py

Writes tests/golden/io/: a float64 tensor (order 3), a mask from the
reference's exact-count sampler, an order-1 tensor, and the metrics CSV the
reference CLI prints for (est, truth, mask).
"""
from __future__ import annotations

import contextlib
import io
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from fctnlr import fileio  # noqa: E402
from fctnlr.cli import main  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "io")


def run():
    os.makedirs(OUT, exist_ok=True)
    rng = np.random.default_rng(7)
    truth = rng.uniform(0, 1, (9, 7, 4))
    est = truth + 0.05 * rng.standard_normal(truth.shape)
    fileio.write_tensor(os.path.join(OUT, "truth.fctn"), truth)
    fileio.write_tensor(os.path.join(OUT, "est.fctn"), est)
    fileio.write_tensor(os.path.join(OUT, "vec.fctn"), np.arange(5.0))
    mask = fileio.sample_mask(truth.shape, 0.3, 11)
    fileio.write_mask(os.path.join(OUT, "mask.fctn"), mask)
    buf = io.StringIO()
    with contextlib.redirect_stdout(buf):
        rc = main(["metrics", "--truth", os.path.join(OUT, "truth.fctn"), "--est", os.path.join(OUT, "est.fctn"),
                   "--mask", os.path.join(OUT, "mask.fctn")])
    assert rc == 0
    with open(os.path.join(OUT, "metrics.csv"), "w") as fh:
        fh.write(buf.getvalue())
    print(buf.getvalue())


if __name__ == "__main__":
    run()
