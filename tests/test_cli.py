"""The CSV/CLI contract (proj/tools/fastdctplus.cpp, bench.hpp:22-372):
descriptor parsing / formatting and CSV rows identical to the reference's
(CPU), and the runners on the GPU producing the reference's row layout, with
the deterministic metrics (prune rate) equal to the reference's."""
import ctypes as C
import subprocess
import sys

import numpy as np
import pytest

from oracle import checkers as O

DESCRIPTORS = ["selfloop:1:1.5", "edge:2:3:1.5", "edge:3:5:-0.7", "selfloop:12:1e-5", "edge:1:1024:2.5e+10",
               "selfloop:1:0.1234567891", " selfloop:1:1.5", "selfloop:0:1", "edge:3:2:1", "edge:1:2",
               "foo:1:2", "selfloop:1:x", "selfloop:1:0", ""]


@pytest.mark.parametrize("text", DESCRIPTORS)
def test_update_descriptors_match_reference(reference, text):
    from paper_2409_08970_b200 import InvalidArgument, cli

    buf = C.create_string_buffer(256)
    rc = reference.lib.ref_format_update(text.encode(), buf, 256)
    if rc == 0:
        assert cli.format_update(cli.parse_update(text)) == buf.value.decode()
    else:
        with pytest.raises(InvalidArgument) as e:
            cli.parse_update(text)
        assert str(e.value) == reference.lib.ref_last_error().decode()


@pytest.mark.parametrize("value", [301.23456789, 0.0, -1.5e-300, 1e300, 12345678.9, float("inf")])
def test_csv_rows_match_reference(reference, value):
    from paper_2409_08970_b200 import cli

    buf = C.create_string_buffer(512)
    reference.lib.ref_csv_row(b"runtime", 64, b"edge:2:3:1.5", b"nmvp", b"ratio_to_dct", value, buf, 512)
    assert cli.csv_row("runtime", 64, "edge:2:3:1.5", "nmvp", "ratio_to_dct", value) == buf.value.decode()
    assert cli.CSV_HEADER == "mode,size,update,method,metric,value\n"


def _rows(text):
    lines = text.strip().split("\n")
    assert lines[0] == "mode,size,update,method,metric,value"
    return [ln.split(",") for ln in lines[1:]]


@pytest.mark.gpu
def test_accuracy_and_runtime_rows():
    from paper_2409_08970_b200 import cli

    cfg = cli.Config(sizes=[8, 64], trials=64)
    rows = _rows(cli.run_accuracy(cfg))
    assert [(r[0], int(r[1]), r[2], r[3], r[4]) for r in rows] == [
        ("accuracy", n, u, "fastdctplus", "mean_snr_db") for n in (8, 64) for u in cfg.updates]
    assert all(float(r[5]) > 200.0 for r in rows)  # structured route vs the dense product
    rows = _rows(cli.run_runtime(cli.Config(sizes=[64], trials=512, updates=["selfloop:1:1.5"])))
    assert [(r[3], r[4]) for r in rows] == [("dct", "mean_ns"), ("fastdctplus", "mean_ns"), ("nmvp", "mean_ns"),
                                           ("fastdctplus", "setup_ns"), ("dct", "ratio_to_dct"),
                                           ("fastdctplus", "ratio_to_dct"), ("nmvp", "ratio_to_dct")]
    assert all(float(r[5]) > 0 for r in rows)


@pytest.mark.gpu
def test_prune_cell_matches_reference_decisions(reference):
    """Same pool (Rng(mix_seed(seed, n, cp))), threshold and branch decisions
    as the reference's measure_prune_cell: the prune rate is identical; the
    coefficients of the pruned branch differ from the direct ones by the
    truncation only."""
    from paper_2409_08970_b200 import calibrate_prune_threshold, cli

    n, cp, seed = 32, 16, 1
    thr = calibrate_prune_threshold(n, 0.99, 0.7, 512, seed)
    r = cli.measure_prune_cell(n, cp, thr, 1e-12, 300, cli.mix_seed(seed, n, cp))
    pool = reference.fill(cli.mix_seed(seed, n, cp), 2, n, 300, 0.99)
    ens = reference.ensemble(n, [O.Update(0, 1.5, 1), O.Update(1, 1.5, 2, 3)], cp, thr)
    _, _, pruned = ens.forward_all_bounds(pool)
    assert r["prune_rate"] == float(np.mean(pruned != 0))
    assert 0.0 < r["selection_agreement"] <= 1.0 and r["psnr_db"] > 0.0
    text = cli.run_prune(cli.Config(sizes=[n], trials=300, cp=cp, threshold=thr))
    metrics = [row[4] for row in _rows(text)]
    assert metrics == ["mean_ns", "mean_ns", "speedup", "mean_mse", "max_mse", "psnr_db", "selection_agreement",
                       "prune_rate", "threshold"]


@pytest.mark.gpu
def test_transform_subcommand_matches_reference(reference):
    s = np.random.default_rng(3).standard_normal(64)
    text = " ".join(f"{v:.17g}" for v in s)
    run = lambda *a: subprocess.run([sys.executable, "-m", "paper_2409_08970_b200.cli", "transform", *a],  # noqa: E731
                                    input=text, capture_output=True, text=True, check=True).stdout
    got = np.array([float(v) for v in run("--update", "edge:3:5:1.5").split()])
    want = reference.plan(64, O.Update(1, 1.5, 3, 5)).forward(s)[0]
    assert O.parity(got[None], want[None]) <= 1e-10
    back = np.array([float(v) for v in
                     subprocess.run([sys.executable, "-m", "paper_2409_08970_b200.cli", "transform", "--update",
                                     "edge:3:5:1.5", "--inverse"], input=" ".join(f"{v:.17g}" for v in got),
                                    capture_output=True, text=True, check=True).stdout.split()])
    assert np.max(np.abs(back - s)) < 1e-10 * np.max(np.abs(s))
    bad = subprocess.run([sys.executable, "-m", "paper_2409_08970_b200.cli", "transform", "--update", "nope"],
                         input=text, capture_output=True, text=True)
    assert bad.returncode == 1 and bad.stderr.startswith("error: bad update descriptor")
